// naive.cuh — decompress-then-count on the device (naive.cu), verification only.
#pragma once
#include "word.cuh"

namespace gt {
// tokens / file_off (host, optional): count these per-file token streams
// (word ids) instead of expanding the grammar — the plain text count
void naive_run(DeviceDag* d, int task, int seq_len, DevRecords* R, int* wbits_out,
               const uint32_t* tokens = nullptr, const uint64_t* file_off = nullptr);
}
