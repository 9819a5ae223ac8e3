// seq.cuh — l-gram tasks (seq.cu).
#pragma once
#include "word.cuh"

namespace gt {
// mode: GT_TOPDOWN (dense per-file weights), GT_TOPDOWN_SPARSE (presence-
// guided sparse weights) or GT_BOTTOMUP (pooled per-rule window tables,
// bottomup.cu; top-down sparse when over the memory budget).  Returns the
// strategy that ran.
int run_sequences(DeviceDag* d, int task, int seq_len, int mode, DevRecords* R, int* wbits_out);
}
