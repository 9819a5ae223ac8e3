/*
 * gtadoc_b200.h — C-ABI of the B200-native analytics-on-compression library
 * (libgtadoc_b200.so).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * What it replaces in the reference (pure-Python package `gtadoc`, paths
 * relative to /root/reference/pkg/src/gtadoc):
 *
 *   gt_open          grammar.py:193-228  deserialize_grammar(data) -> Grammar
 *                    dag.py:131-230      build_dag(grammar) -> Dag
 *                    (plus the level schedule that engine.py:196-227 and
 *                    engine.py:313-335 discover round by round)
 *   gt_run           tasks.py:171-185    run_task(dag, task, cfg, seq_len)
 *                    i.e. tasks.py:122-168 word_count / sort_by_frequency /
 *                    inverted_index / term_vector / sequence_count /
 *                    ranked_inverted_index, and underneath them the kernel
 *                    plugin backend.py:26-46 (_kernels.py:61-309 round kernels)
 *   gt_result_view   the output containers tasks.py:61-88, as compact arrays
 *                    already in the order render() (tasks.py:233-263) prints
 *   gt_last_error    the exception message; the status code selects the
 *                    class of errors.py:11-46 (see gt_status below)
 *
 * The reference's own kernel plugin API (backend.kernels(name) returning a
 * module of 11 numba round functions over host int64 arrays) cannot host a
 * device backend without editing the reference (backend names are validated
 * against auto|numba|python, backend.py:30-31) and would force a host round
 * trip per round, so the boundary sits one level up, at the task entry
 * points, exactly as BASELINE.json north_star prescribes.  The Python facade
 * paper_2106_06889_b200/tasks.py mirrors tasks.py names and containers on top
 * of this ABI; INTEGRATION.md shows the ctypes binding.
 *
 * Threading: a gt_ctx is single-threaded (one CUDA stream on one device).
 * Different contexts (e.g. one per device / rank) may be used concurrently.
 */
#ifndef GTADOC_B200_H
#define GTADOC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GT_ABI_VERSION 3

/* Status codes.  Exception class (errors.py) and CLI exit code in brackets. */
enum gt_status {
  GT_OK = 0,
  GT_E_USAGE = 1,      /* UsageError        [exit 1]  errors.py:15-16 */
  GT_E_RESOURCE = 2,   /* ResourceError     [exit 2]  errors.py:25-28 */
  GT_E_FORMAT = 3,     /* FormatError       [exit 3]  errors.py:31-34 */
  GT_E_CORRUPTION = 4, /* CorruptionError   [exit 3]  errors.py:37-40 */
  GT_E_DEVICE = 5      /* CUDA failure      -> ResourceError [exit 2]  */
};

/* Task ids: tasks.py:47-56 HOOKS order. */
enum gt_task {
  GT_WORDCOUNT = 0,
  GT_SORT = 1,
  GT_INVERTEDINDEX = 2,
  GT_TERMVECTOR = 3,
  GT_SEQCOUNT = 4,
  GT_RANKEDINVERTEDINDEX = 5
};

/* engine.py:31 STRATEGIES (requests).  gt_view.strategy reports what ran:
 * GT_TOPDOWN_SPARSE is the presence-guided sparse per-file top-down pass the
 * library uses where the reference goes bottom-up for many files. */
enum gt_strategy { GT_AUTO = 0, GT_TOPDOWN = 1, GT_BOTTOMUP = 2, GT_TOPDOWN_SPARSE = 3 };

typedef struct gt_ctx gt_ctx;
typedef struct gt_result gt_result;

/* Corpus / DAG statistics (SURVEY.md §8 notation). */
typedef struct gt_info {
  uint64_t num_words;      /* V  = dictionary.num_words                       */
  uint64_t num_splitters;  /*      dictionary.num_splitters                   */
  uint64_t num_rules;      /* R                                              */
  uint64_t num_files;      /* F  = len(dag.segments)                          */
  uint64_t total_elements; /* E  = dag.total_elements                         */
  uint64_t root_len;       /* L0                                              */
  uint64_t sub_pairs;      /* E_sub = len(dag.sub_ids)                        */
  uint64_t own_pairs;      /* E_own = len(dag.own_ids)                        */
  uint64_t words;          /* W  = exp_len[0] (uncompressed-equivalent words) */
  int64_t depth;           /* dag.depth = height of the root                  */
  int64_t td_levels;       /* top-down levels (= reference top-down rounds)   */
  int64_t bu_levels;       /* bottom-up levels (= reference bottom-up rounds) */
  uint64_t device_bytes;   /* device memory held by the context               */
  double init_ms;          /* gt_open wall time (the "initialization" phase)  */
  uint64_t td_edges;       /* non-root parent edges (top-down pass items)     */
  uint64_t load_flags;     /* bit 0: rule chain parsed in the chunked form;   */
                           /* bit 1: per-file cells held in u32 (files < 2^32 words); */
                           /* bit 2: word count / inverted index run over the  */
                           /* single-parent contraction (heads only)           */
} gt_info;

/*
 * Result view.  Arrays are owned by the gt_result (host memory) and stay
 * valid until gt_result_free.  Layout per task:
 *
 *  WORDCOUNT  n records (id = word, count), ascending word id.
 *  SORT       n records (id = word, count), (-count, word) order.
 *  INVERTEDINDEX  n_groups words (group_id = word, ascending); records
 *             group_off[g]..group_off[g+1] hold id = file (ascending).
 *             count == NULL.
 *  TERMVECTOR n_groups = F files; records of file f are group_off[f].. with
 *             (id = word, count) in (-count, word) order.
 *  SEQCOUNT   n_groups = F files; records of file f: gram + count in
 *             (-count, gram) order.  wbits > 0: gram packed big-endian in
 *             key[i] (wbits bits per word, sequence.py:229-256); wbits == 0
 *             (gram mode, seq_len*wbits > 63): gram[i*seq_len + j].
 *  RANKEDINVERTEDINDEX  n_groups grams in ascending gram order (group_key or
 *             group_gram); records of gram g: (id = file, count) in
 *             (-count, file) order.
 */
typedef struct gt_view {
  int32_t task;
  int32_t seq_len;
  int32_t wbits;
  int32_t strategy; /* the concrete strategy that ran (GT_TOPDOWN/GT_BOTTOMUP) */
  uint64_t n_groups;
  const uint64_t* group_off;  /* n_groups + 1 entries, or NULL */
  const uint32_t* group_id;   /* II: word id per group */
  const uint64_t* group_key;  /* RII packed gram per group */
  const uint32_t* group_gram; /* RII gram mode: seq_len words per group */
  uint64_t n;                 /* records */
  const uint32_t* id;         /* word id or file id per record */
  const uint64_t* key;        /* SC packed gram per record */
  const uint32_t* gram;       /* SC gram mode: seq_len words per record */
  const uint64_t* count;      /* per record; NULL for INVERTEDINDEX */
  /* timings of this run */
  double device_ms; /* device time of the traversal + assembly kernels      */
  double d2h_ms;    /* device->host copy of the compact result              */
  double total_ms;  /* wall time of gt_run                                  */
  uint64_t d2h_bytes;
  uint64_t kernel_launches; /* kernels launched by this gt_run              */
  /* (ABI 2) narrow copies: when every record offset fits 32 bits the group
   * offsets travel as u32 (group_off == NULL, group_off32 set), and when the
   * task's counts are bounded below 2^32 (per-file counts: the longest file;
   * corpus counts: W) so do the counts (count == NULL, count32 set) — a
   * third less PCIe traffic for the count-carrying results */
  const uint32_t* count32;
  const uint32_t* group_off32;
  /* (ABI 3) narrow ids: when every record id is below 2^8 or 2^16 (file ids
   * of an inverted index / ranked inverted index on <= 256 / 65536 files,
   * word ids of a vocabulary that small) the ids travel id_bytes (1 or 2)
   * wide in id_narrow and id == NULL; otherwise id_narrow == NULL, id_bytes == 4 */
  const void* id_narrow;
  int32_t id_bytes;
  int32_t reserved_;
} gt_view;

int gt_abi_version(void);
const char* gt_last_error(void); /* message of the last failing call on this thread */

/* Parse + validate GTDC bytes, build the device DAG and level schedule on
 * CUDA device `device`.  file_lo/file_hi restrict per-file work and root
 * segments to files [file_lo, file_hi) (multi-GPU sharding);
 * pass 0, UINT64_MAX for the whole corpus. */
int gt_open(const uint8_t* gtdc, size_t nbytes, int device, uint64_t file_lo,
            uint64_t file_hi, gt_ctx** out);
int gt_info_get(const gt_ctx* ctx, gt_info* out);

/* Run one analytics task (tasks.py:171-185).  strategy: gt_strategy;
 * file_set_width: TraversalConfig.file_set_width (engine.py:39, default 64).
 * seq_len is used by SEQCOUNT / RANKEDINVERTEDINDEX only. */
int gt_run(gt_ctx* ctx, int task, int seq_len, int strategy, int file_set_width,
           gt_result** out);
/* Run several tasks over one DAG in one call; outs[i] receives the result of
 * tasks[i] (the same result gt_run would give).  Tasks that share a traversal
 * share it on the device: a WORDCOUNT (or SORT) together with an
 * INVERTEDINDEX whose owned files fit one presence word (<= 64) and that runs
 * top-down run as ONE top-down pass over {weight, presence} rule pairs — the
 * level chain, word reduce and compaction of both tasks in one launch (the
 * bench step: BASELINE.json's word count + inverted index).  The shared pass's
 * device time is charged to the word-count result (the inverted index's
 * device_ms is 0); the other tasks run as by gt_run.  On error every outs[i]
 * is NULL. */
int gt_run_many(gt_ctx* ctx, const int* tasks, int ntasks, int seq_len, int strategy,
                int file_set_width, gt_result** outs);
int gt_result_view(const gt_result* res, gt_view* out);
void gt_result_free(gt_result* res);
void gt_close(gt_ctx* ctx);

/* Decompress-then-count on the device: the reference's naive counterparts
 * (oracle_task, tasks.py:191-227; oracle.py:19-60) — expand the grammar to
 * the token stream and count plainly — as an independent ground truth at
 * corpus sizes the CPU oracles cannot hold.  Same result
 * layout as gt_run; verification only (gt_run never uses it).  Sequence
 * tasks need packed grams (seq_len * wbits <= 63). */
int gt_run_naive(gt_ctx* ctx, int task, int seq_len, gt_result** out);

/* The plain-text counterpart of gt_run_naive, for `verify` on an input
 * directory (cli.py:137-147): count the given per-file token streams (word
 * ids, file f = tokens[file_off[f] .. file_off[f+1]), nfiles == num_files,
 * e.g. from gt_tokenize of the files the grammar was compressed from) with
 * the same device counting and ordering stage — no grammar expansion and no
 * use of the loaded DAG's arrays, so it checks the loader too.  Same result
 * layout as gt_run; verification only. */
int gt_count_tokens(gt_ctx* ctx, int task, int seq_len, const uint32_t* tokens, const uint64_t* file_off,
                    uint64_t nfiles, gt_result** out);

/* Multi-GPU sharding: restrict per-file work and root seeds of
 * subsequent gt_run calls to files [file_lo, file_hi) (clamped to F); the
 * DAG itself is replicated in every context. */
int gt_set_files(gt_ctx* ctx, uint64_t file_lo, uint64_t file_hi);

/* WORDCOUNT / SORT result from a dense u64[num_words] DEVICE vector on the
 * context's device (e.g. the NCCL all-reduce of every shard's
 * gt_device_word_counts): the assembly half of gt_run. */
int gt_assemble_counts(gt_ctx* ctx, int task, const uint64_t* dev_counts, gt_result** out);

/* Replicate a loaded context onto `device`: the DAG is built
 * once and copied peer-to-peer (NVLink) to the other GPUs, replacing one
 * host upload + device build (dag.py:131-230) per GPU.  The copy keeps the
 * source's file range; shard it with gt_set_files.  Same device is allowed
 * (several shards of one corpus on one GPU). */
int gt_clone(const gt_ctx* src, int device, gt_ctx** out);

/* Number of visible CUDA devices (0 when none). */
int gt_device_count(void);

/* Sum the dense word counts left by the last WORDCOUNT/SORT run of every
 * context in srcs (file-range shards of one corpus, on any devices) into
 * dst's device: one kernel on dst's device reads each shard's
 * u64[num_words] vector in place through peer memory (NVLink) — the
 * all-reduce of SURVEY §8e fused into the gather, no staging copy — and
 * leaves the exact integer totals as dst's gt_device_word_counts (then
 * gt_assemble_counts gives the corpus-wide result).  dst may be one of
 * srcs. */
int gt_sum_word_counts(gt_ctx* dst, gt_ctx* const* srcs, int n);

/* Dense global word counts left on the device by the last WORDCOUNT/SORT run
 * (u64[num_words]); for NCCL all-reduce across shards.  Returns the device
 * pointer or NULL. */
uint64_t* gt_device_word_counts(gt_ctx* ctx);

/* Test/diagnostic export of a DAG array as int64 (same content as the
 * reference Dag field): name in {own_ids, own_freqs, own_off,
 * own_token_count, sub_ids, sub_freqs, sub_off, par_ids, par_freqs, par_off,
 * num_in_edge, num_out_edge, root_freq, exp_len, segments, td_level,
 * bu_level, weight}; device-layout diagnostics: tid (the top-down row of
 * every rule), cont_head / cont_mult / cont_level / cont_row (the
 * single-parent contraction in tid space: head tid, multiplier, contracted
 * level, head row; building it if needed; empty when a multiplier outgrew
 * 32 bits) and cont_sizes ([heads, head edges, levels] of a built
 * contraction, else empty).  Returns the element count (call with out=NULL
 * to size), or -1 on error. */
int64_t gt_dag_array(gt_ctx* ctx, const char* name, int64_t* out, int64_t cap);

/* Per-kernel timing: while enabled, every kernel launched by this thread is
 * bracketed by CUDA events on its stream.  gt_profile_report writes
 * "name\tlaunches\ttotal_ms\n" lines (aggregated by kernel name, since the
 * last report) into buf and returns the length needed (or -1); the report
 * is consumed only by a call with buf != NULL.  ctx may be NULL (profile a
 * gt_open: enable before it, report after it). */
int gt_profile(gt_ctx* ctx, int enable);
int64_t gt_profile_report(gt_ctx* ctx, char* buf, size_t cap);

/* Test hook of the pooled hash tables' insert path (bottomup.cu), the
 * analogue of the reference's add_batch stress kernel (_kernels.py:117-126,
 * pkg/tests/test_table.py:145-164): n concurrent (key, delta) inserts into
 * one open-addressing table of `capacity` (power of two) slots on `device`;
 * copies back the slot arrays (empty key = 0xFFFFFFFF).  GT_E_RESOURCE when
 * the table overflowed (the reference's FULL status). */
int gt_table_add_batch(int device, const uint32_t* keys, const uint64_t* deltas, uint64_t n,
                       uint32_t capacity, uint32_t* out_keys, uint64_t* out_counts);

/* Evict L2 (writes a buffer larger than L2 on the context's stream). */
int gt_flush_l2(gt_ctx* ctx);
/* Synchronize the context's stream. */
int gt_sync(gt_ctx* ctx);

/* ---- native rendering (host only; works without a GPU) -------------------
 * Byte-identical to tasks.py:233-263 render(); the SHA-256 of the rendering
 * is the reference CLI manifest's outputDigest (cli.py:121-133).  A gt_dict
 * holds the word strings of a GTDC blob (grammar.py:193-228 layout). */
typedef struct gt_dict gt_dict;
int gt_dict_open(const uint8_t* gtdc, size_t nbytes, gt_dict** out);
void gt_dict_close(gt_dict* dict);
/* render a result view (gt_result_view, or arrays built by the caller);
 * *text is malloc'd, NUL-terminated, released with gt_free_text */
int gt_render_view(const gt_dict* dict, const gt_view* view, char** text, uint64_t* len);
void gt_free_text(char* text);
/* SHA-256 of the rendering without materialising it; *len = its byte count */
int gt_digest_view(const gt_dict* dict, const gt_view* view, uint8_t sha256[32], uint64_t* len);
int gt_sha256(const void* data, uint64_t nbytes, uint8_t out[32]);

/* ---- native compressor (host only) ------------------------------------------
 * Ingest (ingest.py:30-121: strict UTF-8, Python str.split() whitespace,
 * first-appearance word ids, one splitter after each file) + Sequitur
 * (sequitur.py:46-258, lowest-free rule ids) + GTDC serialization
 * (grammar.py:164-174): the same bytes as the reference's compress command.
 * files[i] / lens[i]: the corpus files in order.  *out is malloc'd (release
 * with gt_compress_free).  stats (optional, 4 entries): files, rules, words,
 * stream symbols.  Status 101 = invalid UTF-8 (IngestError; stats[0] = the
 * file index, gt_compress_last_error has the byte offset). */
int gt_compress(const uint8_t* const* files, const uint64_t* lens, uint64_t nfiles, uint8_t** out,
                uint64_t* out_len, uint64_t* stats);
void gt_compress_free(uint8_t* p);
const char* gt_compress_last_error(void);
/* The ingest half alone: the files as word-id token streams (the ids
 * gt_compress gives the same files), file f = tokens[file_off[f] ..
 * file_off[f+1]) (file_off: nfiles + 1 entries, caller-allocated).
 * *tokens is malloc'd (release with gt_compress_free). */
int gt_tokenize(const uint8_t* const* files, const uint64_t* lens, uint64_t nfiles, uint32_t** tokens,
                uint64_t* file_off);

#ifdef __cplusplus
}
#endif
#endif /* GTADOC_B200_H */
