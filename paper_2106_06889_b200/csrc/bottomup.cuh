// bottomup.cuh — the bottom-up strategy with pooled hash tables (bottomup.cu).
#pragma once
#include "word.cuh"

namespace gt {

// Global word counts (dense u64[V]) from the per-rule tables; false when the
// arena would exceed `budget` bytes (the caller falls back to top-down).
bool bu_word_counts(DeviceDag* d, DBuf& counts, u64 budget);

// Term vector (task = GT_TERMVECTOR) or inverted index (GT_INVERTEDINDEX)
// from per-file tables merged from the per-rule tables; false = over budget.
bool bu_file_tables(DeviceDag* d, int task, DevRecords* R, u64 budget);

// Bottom-up l-gram cells (seq.cu): per-rule window tables merged children-
// first, then per-file tables; (run, file, count) cells in (run, file) order.
// run/src: the sorted window occurrences (gram run id, rule id or R + owned
// segment).  false = over budget.
bool bu_seq_cells(DeviceDag* d, u32 l, const u32* run, const u32* src, u64 N, u64 nruns, DBuf& crun, DBuf& ccol,
                  DBuf& ccnt, u64* n_out, u64 budget);

// helpers from word.cu: root words of the owned segments into a dense u64[V];
// root reference counts of the owned segments per rule (u64[R])
void bu_root_words_dense(DeviceDag* d, u64* out);
void td_root_seeds(DeviceDag* d, u64* row);

// add_batch test hook (see gt_table_add_batch)
int table_add_batch(int device, const u32* keys, const u64* deltas, u64 n, u32 cap, u32* out_keys,
                    u64* out_vals);

// device bytes the task paths may use (free device memory + unused pool)
u64 scratch_budget(const DeviceDag* d);

}  // namespace gt
