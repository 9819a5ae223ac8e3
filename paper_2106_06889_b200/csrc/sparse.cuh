// sparse.cuh — presence-guided sparse per-file weights (sparse.cu).
#pragma once
#include "word.cuh"

namespace gt {

// (rule, file) pairs with nonzero per-file weight, CSR by rule, files
// (relative to file_lo) ascending within a rule
struct SparseW {
  DBuf off;   // u64[R+1]
  DBuf file;  // u32[P]
  DBuf wt;    // u64[P]
  u64 P = 0;
};

// rows of bitsets -> CSR: row r's words at bits[r*rs_row + j*rs_col]
// (j < FW); off u64[nrows+1], col = col_base + set-bit index, ascending;
// optional row id per pair and per-row counts.  Returns the pair count.
u64 bits_to_csr(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, DBuf& off, DBuf& col,
                DBuf* row_of, cudaStream_t st, u32 col_base = 0, DBuf* row_cnt = nullptr);

// the two halves of bits_to_csr (count + scan, then expansion once the
// caller knows P = off[nrows]) for callers that batch their host syncs
void bits_count(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, DBuf& off, DBuf& cnt,
                cudaStream_t st);
void bits_groups(const u64* bits, u64 nrows, u32 FW, u32 col_base, DBuf& files, DBuf& gid, DBuf& goff, u64* n_out,
                 u64* ng_out, cudaStream_t st);
void bits_expand(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, const DBuf& off, u64 P,
                 DBuf& col, DBuf* row_of, cudaStream_t st, u32 col_base = 0);

// presence pass + pairs + weights; optionally hands back the word presence
// bitsets u64[FW][V] of the same pass
void sparse_file_weights(DeviceDag* d, SparseW* s, DBuf* word_pres, u32* FW);

// term vector for many files (render order: file, -count, word)
void sparse_term_vector(DeviceDag* d, DevRecords* R);

// gram occurrences (run id, source) -> reduced (run << FB | file, count)
// cells in (run, file) order; returns the cell count
u64 sparse_run_cells(DeviceDag* d, const SparseW& s, const u32* rid, const u32* src, u64 N, int FB,
                     DBuf& cell_key, DBuf& cell_cnt);

}  // namespace gt
