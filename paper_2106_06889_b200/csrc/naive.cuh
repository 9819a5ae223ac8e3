// naive.cuh — decompress-then-count on the device (naive.cu), verification only.
#pragma once
#include "word.cuh"

namespace gt {
void naive_run(DeviceDag* d, int task, int seq_len, DevRecords* R, int* wbits_out);
}
