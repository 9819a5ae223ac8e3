// seq.cuh — l-gram tasks (seq.cu).
#pragma once
#include "word.cuh"

namespace gt {
void run_sequences(DeviceDag* d, int task, int seq_len, bool sparse, DevRecords* R, int* wbits_out);
}
