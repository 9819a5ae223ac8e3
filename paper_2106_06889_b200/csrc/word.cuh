// word.cuh — word-task drivers (word.cu) and device result records.
#pragma once
#include "gt_internal.cuh"

namespace gt {

// Compact device-side result (render order) before the D2H copy.
struct DevRecords {
  u64 n = 0, n_groups = 0;
  DBuf group_off, group_id, group_key, group_gram;  // u64, u32, u64, u32
  DBuf id, key, gram, count;                        // u32, u64, u32, u64
  // u32 forms written by the producing kernel itself (the D2H skips the
  // narrowing launch); valid only when the flag is set
  DBuf count32, group_off32;
  bool count32_ok = false, group_off32_ok = false;
  DBuf id_narrow;   // ids id_bytes (1 / 2) wide, written by the producing kernel
  int id_bytes = 4; // 4: no narrow copy
};

void td_word_counts(DeviceDag* d, DBuf& counts);
void td_file_counts(DeviceDag* d, DBuf& counts, bool* is32);
bool td_word_records(DeviceDag* d, DevRecords* R);
bool td_presence_records(DeviceDag* d, DevRecords* R);
// done (optional): recorded on the stream once the device work is queued —
// before the host waits for the record totals, so that an event pair around
// the call times the device, not the host's wake-up
bool td_wc_ii_records(DeviceDag* d, DevRecords* wc, DevRecords* ii, cudaEvent_t done = nullptr);
void order_by_count(DeviceDag* d, DevRecords* R, u32 ncols, const u32* file);
void td_file_presence(DeviceDag* d, DBuf& pres, u32* FW, DBuf* rows_out = nullptr);
// heads: the contraction's head rows when it is in use (*contracted set; the
// caller maps a rule's tid t to row c_tid[c_hd[t]] with multiplier c_ml[t])
void td_file_weights(DeviceDag* d, DBuf& w, u32* C, bool* is32, bool heads = false, bool* contracted = nullptr);
void assemble_counts(DeviceDag* d, const void* dense, u64 V, u32 ncols, bool by_count, DevRecords* R,
                     bool dense32 = false);
void assemble_presence(DeviceDag* d, const u64* pres, u32 FW, DevRecords* R);

}  // namespace gt
