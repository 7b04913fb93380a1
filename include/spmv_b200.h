/*
 * spmv_b200.h — C ABI of the B200-native SpMV engine (libspmv_b200.so).
 *
 * Every entry point replaces one function of the reference package
 * `spmvkit` (pure Python/numpy, /root/reference/pkg/src/spmvkit); the
 * replaced interface is cited as file:line next to each declaration.
 *
 * Conventions
 *   - Plain C types only: device pointers, 64-bit sizes, an opaque
 *     `void* stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Indices are the reference's uint32 (formats.py:24), DIA offsets its
 *     int32 (formats.py:25).  Values are f32 or f64 (formats.py:27).
 *   - DIA values are the reference's row-major (padded_rows, ndiags) block
 *     (formats.py:166-207), padded_rows a multiple of ROW_PAD = 8.
 *   - Every call returns an spmv_status; spmv_last_error() gives the
 *     thread-local message of the last failing call.  The codes map 1:1 to
 *     the reference's exception classes (errors.py:4-37).
 *   - SpMV calls never write caller memory other than y (kernels.py:59,72,
 *     94: the kernel owns a fresh y).  Workspace lives in the plan objects.
 *     Every entry point is reentrant, also on one plan (kernels
 *     are pure; bench.py:167-172 calls kernels from several threads): the
 *     per-launch scratch of a plan (partial-sum slots, the warp-stream range
 *     counter) is kept per CUDA stream — allocated, zero-filled, on the
 *     first launch on a stream and reused after — so products on different
 *     streams with disjoint outputs may run concurrently.  Lazily built
 *     parts (vla row lists, the host-pipeline staging) are built once under
 *     the plan's lock; host-pipeline calls on one plan are serialised on the
 *     device (each waits for the previous one's end).
 *   - Calls that return a host-visible count (plan creation, conversion
 *     analyze steps) synchronise `stream`; SpMV calls are asynchronous.
 */
#ifndef SPMV_B200_H
#define SPMV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMV_B200_ABI_VERSION 2

typedef enum {
    SPMV_F32 = 0,
    SPMV_F64 = 1
} spmv_dtype;

typedef enum {
    SPMV_OK = 0,
    SPMV_DIMENSION_MISMATCH = 1,   /* errors.py:8  DimensionMismatch      */
    SPMV_UNSORTED_INPUT = 2,       /* errors.py:12 UnsortedInput          */
    SPMV_FILL_RATIO_EXCEEDED = 3,  /* errors.py:16 FillRatioExceeded      */
    SPMV_UNSUPPORTED = 4,          /* errors.py:20 UnsupportedCombination */
    SPMV_CUDA_ERROR = 5,
    SPMV_INVALID_ARG = 6,
    SPMV_INDEX_OVERFLOW = 7        /* errors.py:36 IndexOverflow          */
} spmv_status;

/* ---- library ----------------------------------------------------------- */
int spmv_abi_version(void);
const char* spmv_last_error(void);
/* Number of SMs of the current device (grid sizing; 148 on B200). */
int spmv_device_sm_count(int* out);

/* ---- plan configuration ------------------------------------------------- */
/* Kernel choices of one plan.  Every field at its "auto" value (0, or -1
 * where noted) keeps the plan's measured default, which depends on the
 * row-length histogram.  A plan's configuration is fixed at creation, so
 * several plans of one matrix can run different kernels side by side in
 * one process; the run-first tuner (autotune.py:60-139, hpcg.py:270-304:
 * "format plus CSR bin thresholds") creates one plan per candidate and
 * times them.  Replaces the process-global environment switches of ABI 1. */
#define SPMV_PLAN_CONFIG_VERSION 1
typedef struct {
    int32_t version;          /* SPMV_PLAN_CONFIG_VERSION                            */
    int32_t tile;             /* entries per TMA tile (CSR: 1024 1664 2048 2304 4096; */
                              /* COO: 1024 1536 2048); 0 = plan's choice              */
    int32_t groups;           /* consumer groups per tile CTA (CSR 1/3/4, COO 1/6/7); */
                              /* 0 = plan's choice; unknown combinations fall back    */
    int32_t exact_len;        /* CSR warp-stream kernel: rows of <= exact_len entries */
                              /* are never split between warp ranges and are summed  */
                              /* left to right (bit-exact), 1..32; 0 = 32.  The tile  */
                              /* kernels always use 32 (their tile extension)         */
    int32_t warp_stream;      /* whole-matrix kernel: -1 plan's choice (warp-stream   */
                              /* when rows/runs exceed exact_len), 0 tiles, 1 ws      */
    int32_t ranges_per_warp;  /* warp-stream entry ranges per resident warp 1..64;    */
                              /* 0 = 8                                                */
    int32_t tma_hint;         /* L2 evict_first on the TMA matrix stream: -1 plan's   */
                              /* choice (COO always, CSR with long rows), 0, 1        */
    int32_t ctas_per_sm;      /* cap on resident CTAs per SM; 0 = occupancy limit     */
    int32_t dia_kernel;       /* DIA (groups, stages, threads) 0..4; -1 = auto        */
    int32_t dia_rows;         /* DIA rows per tile, multiple of 8; 0 = auto           */
    int32_t flags;            /* experiments: bit0 products mode, bit1 warp per long  */
                              /* segment (tile kernels); bit2: the panel path's short */
                              /* rows start from +0.0 (np.add.at order; COO plans set */
                              /* it for their CSR view); 0 = off                      */
    int32_t panels;           /* CSR column-panel path for long rows: -1 auto (rows   */
                              /* over 32 entries hold >= half the entries, ncols >=   */
                              /* 65536), 0 off, 1 on (needs col_indices and values at */
                              /* plan creation)                                       */
    int32_t reserved[4];
} spmv_plan_config;

/* Fill *cfg with the auto values (version set).  Plans created with a NULL
 * configuration use exactly these. */
int spmv_plan_config_init(spmv_plan_config* cfg);

/* ---- CSR (kernels.py:69-82 spmv_csr_plain, :143-171 spmv_csr_vla) ------ */
typedef struct spmv_csr_plan spmv_csr_plan;

/* spmv_csr_plan_create with an explicit configuration (NULL = auto; the
 * exact_len argument of spmv_csr_plan_create is cfg->exact_len here) and
 * optionally the matrix's column indices and values (may be NULL).  With
 * them, a matrix whose long rows (over 32 entries) hold most of the
 * entries gets the column-panel path: the plan keeps a panel-major copy of
 * the long rows (csrc/panel.cuh) and whole-matrix products called with the
 * same two arrays read that copy; the arrays must not change afterwards
 * (containers are immutable).  Products called with other
 * arrays run the warp-stream kernel. */
int spmv_csr_plan_create_ex(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                            const uint32_t* row_pointers,
                            const uint32_t* col_indices, const void* values,
                            const spmv_plan_config* cfg, void* stream,
                            spmv_csr_plan** out);
/* The configuration the plan resolved: tile, groups, warp_stream (0/1),
 * ranges_per_warp, tma_hint (0/1) and exact_len as the kernels run them. */
int spmv_csr_plan_config(const spmv_csr_plan* plan, spmv_plan_config* out);

/* Analyse the matrix once: long-row census (rows > exact_len entries), tile
 * size and consumer groups per CTA (G groups share a G+1 stage ring:
 * 1024 x 3 with long rows; else 2304 (2048 below 64M entries) x 3, or
 * 1664 x 4 for rows averaging < 16 entries), the row range of every tile
 * and the list of
 * long rows spanning tiles.  The SpMV kernel streams
 * fixed entry tiles with TMA bulk copies; rows of <= exact_len entries are
 * summed left to right by one thread (bit-exact with spmv_csr_plain); longer
 * rows are reduced in 256-entry vla-32 units (bit-exact with
 * spmv_csr_vla(32) for rows of <= 256 entries inside one tile, deterministic
 * and within 1e-12 otherwise).  exact_len <= 0 selects the default (32). */
int spmv_csr_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                         const uint32_t* row_pointers, int exact_len,
                         void* stream, spmv_csr_plan** out);
int spmv_csr_plan_destroy(spmv_csr_plan* plan);
/* Profiling builds only (-DSPMV_PHASE_TIMING): per-phase cycle counters of
 * the CSR tile kernel, read and reset (8 entries); else SPMV_UNSUPPORTED. */
int spmv_debug_csr_phases(unsigned long long* out8);
/* Debug builds only (-DSPMV_DEBUG_CHECKS): device-side check counters, read
 * and reset — [0] TMA-staged tile/step differs from global memory (a ring
 * race), [1] index out of range, [2] x panel differs from x, [3] other;
 * else SPMV_UNSUPPORTED. */
int spmv_debug_check_counts(unsigned long long* out4);
/* n_long_rows: rows longer than exact_len; n_items: entries per tile;
 * launches: kernels one spmv_csr call launches (1; +1 for the span
 * fix-up of rows split between tiles or warp-stream ranges). */
int spmv_csr_plan_info(const spmv_csr_plan* plan, int64_t* n_long_rows,
                       int64_t* n_items, int64_t* launches);
/* Consumer groups per tile CTA the plan chose (spmv_plan_config.groups). */
int spmv_csr_plan_groups(const spmv_csr_plan* plan, int* groups);
/* spmv_csr with a gap in y: rows >= y_split are stored at y[row + y_gap].
 * A rank's two boundary planes (its first and last halo-reading rows, one
 * CSR matrix) then run in one launch after the halo exchange while y keeps
 * the slab's row order.  Plans without rows over exact_len only
 * (SPMV_UNSUPPORTED otherwise); always runs the tile kernel. */
int spmv_csr_gapped(const spmv_csr_plan* plan, const uint32_t* row_pointers,
                    const uint32_t* col_indices, const void* values,
                    const void* x, int64_t col_base, int64_t x_len, void* y,
                    int64_t y_split, int64_t y_gap, void* stream);
/* Whole-matrix kernel the plan chose: warp_stream = 1 for the warp-stream
 * kernel (matrices with rows longer than exact_len: one contiguous entry
 * range per resident warp, nwarps of them), 2 for the column-panel path
 * (nwarps = panel CTAs x 32), 0 for the tile kernel.  Tile
 * ranges (spmv_csr_range, spmv_csr_host) always use the tile kernel.
 * spmv_plan_config.warp_stream = 0/1 overrides the choice. */
int spmv_csr_plan_path(const spmv_csr_plan* plan, int* warp_stream, int64_t* nwarps);

/* y[r] = sum_j av[j] * x[aj[j] - col_base] over row r.  x holds the window
 * of global columns [col_base, col_base + x_len).  For a single-device
 * product col_base = 0 and x_len = ncols. */
int spmv_csr(const spmv_csr_plan* plan, const uint32_t* row_pointers,
             const uint32_t* col_indices, const void* values, const void* x,
             int64_t col_base, int64_t x_len, void* y, void* stream);

/* Tile-range launches (pipelined host transfers): the plan's tiles are
 * independent except for long rows spanning tiles, which the fix-up adds
 * (fixup = 1 on the last range).  After tiles [0, k) ran, rows
 * [0, row_lo[k]) of y are final; tiles [a, b) read x only below
 * max(maxcol[a..b)) + 1.  spmv_csr_plan_tile_info copies row_lo (ntiles+1)
 * and maxcol (ntiles) to host arrays (maxcol is computed on first use). */
int spmv_csr_plan_tiles(const spmv_csr_plan* plan, int64_t* ntiles,
                        int64_t* tile);
int spmv_csr_plan_tile_info(spmv_csr_plan* plan,
                            const uint32_t* col_indices,
                            uint32_t* row_lo_host, uint32_t* maxcol_host,
                            void* stream);
int spmv_csr_range(const spmv_csr_plan* plan, const uint32_t* row_pointers,
                   const uint32_t* col_indices, const void* values,
                   const void* x, int64_t col_base, int64_t x_len, void* y,
                   int64_t tile_begin, int64_t tile_end, int fixup,
                   void* stream);

/* Host x -> host y (see "host-buffer products" below; the plan owns the
 * pipe): x goes up in chunks that ramp up to ncols / chunks columns (at
 * least 1M) and down again at the end; each tile range runs once the x it
 * reads has arrived (plans whose whole-matrix kernel is the panel or
 * warp-stream kernel run it once x is complete).  chunks <= 0 = 16. */
int spmv_csr_host(spmv_csr_plan* plan, const uint32_t* row_pointers,
                  const uint32_t* col_indices, const void* values,
                  const void* x_host, void* y_host, int chunks, void* stream);

/* ---- host-buffer products (hostpipe.cuh) ------------------------------- */
/* The reference's calling convention: x in host memory, a fresh y in host
 * memory (kernels.py:46-53, :59, :72, :94).  x goes up in column chunks on
 * a copy stream, each part of the product runs as soon as the x prefix it
 * reads has arrived, finished rows of y come down on a second copy stream.
 * Pinned x is copied directly; pageable x is staged through a pinned ring
 * by host threads.  Pinned y overlaps its copies (pageable y is correct but
 * not overlapped).  Asynchronous: y_host is valid once `stream` is
 * synchronised.  One pipe (the CSR / COO plan's own, or an spmv_host_pipe)
 * runs one call at a time; calls on it are serialised.  chunks <= 0 = 16. */
typedef struct spmv_host_pipe spmv_host_pipe;
typedef struct spmv_coo_plan spmv_coo_plan;
int spmv_host_pipe_create(spmv_host_pipe** out);
int spmv_host_pipe_destroy(spmv_host_pipe* pipe);
/* COO: x chunks up, the whole product, y down. */
int spmv_coo_host(spmv_coo_plan* plan, const uint32_t* row_indices,
                  const uint32_t* col_indices, const void* values,
                  const void* x_host, void* y_host, int chunks, void* stream);
/* DIA: row blocks as soon as x holds row + max_offset (the largest offset,
 * >= 0 if any diagonal is above the main one). */
int spmv_dia_host(spmv_host_pipe* pipe, int dtype, int64_t nrows, int64_t ncols,
                  int64_t ndiags, int64_t padded_rows, const int32_t* offsets,
                  int64_t max_offset, const void* values, const void* x_host,
                  void* y_host, int chunks, const spmv_plan_config* cfg,
                  void* stream);

/* Sub-warp vector kernel, lane l accumulates entries s+l, s+l+L, ... then a
 * pairwise-halving tree over next_pow2(L) lanes: bit-exact with
 * spmv_csr_vla(LaneConfig(L)) (lanes.py:101-128).  1 <= lanes <= 1024. */
int spmv_csr_vla(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                 const uint32_t* row_pointers, const uint32_t* col_indices,
                 const void* values, const void* x, int64_t col_base,
                 int64_t x_len, void* y, int lanes, void* stream);
/* Same, with the CSR plan of the matrix: its long-row census lets the call
 * skip the long-row pass when no row can need it, and rows over 256 entries
 * take a two-phase path (products gathered by all warps, then one ordered
 * fold per row) whose row list and product buffer the plan keeps (built on
 * the first call; not reentrant per plan). */
int spmv_csr_vla_planned(spmv_csr_plan* plan, const uint32_t* row_pointers,
                         const uint32_t* col_indices, const void* values,
                         const void* x, int64_t col_base, int64_t x_len, void* y,
                         int lanes, void* stream);

/* ---- COO (kernels.py:56-66 spmv_coo_plain, :104-140 spmv_coo_vla) ------ */
typedef struct spmv_coo_plan spmv_coo_plan;

/* Checks the row order once.  If rows are not non-decreasing, the plan
 * keeps a stable row-sorted copy of the triples (np.add.at accumulates in
 * storage order per row, kernels.py:65, and a stable sort keeps that
 * order).  Also run-length-encodes the rows (vla kernel, long-run census). */
int spmv_coo_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                         const uint32_t* row_indices,
                         const uint32_t* col_indices, const void* values,
                         void* stream, spmv_coo_plan** out);
int spmv_coo_plan_create_ex(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                            const uint32_t* row_indices,
                            const uint32_t* col_indices, const void* values,
                            const spmv_plan_config* cfg, void* stream,
                            spmv_coo_plan** out);
int spmv_coo_plan_destroy(spmv_coo_plan* plan);
/* Resolved configuration (exact_len is 32 for COO). */
int spmv_coo_plan_config(const spmv_coo_plan* plan, spmv_plan_config* out);
/* row_sorted: 1 when the input rows were already non-decreasing;
 * n_items: entries per tile. */
int spmv_coo_plan_info(const spmv_coo_plan* plan, int64_t* n_runs,
                       int64_t* n_long_runs, int64_t* n_items,
                       int* row_sorted, int64_t* launches);
/* Consumer groups per tile CTA the plan chose (spmv_plan_config.groups). */
/* Whole-matrix kernel the COO plan chose: warp_stream = 0 the COO tile
 * kernel, 1 the warp-stream kernel (runs longer than 32 entries), 2 / 3 a
 * CSR view of the plan's row-sorted triples (row pointers built at plan
 * creation; products read 4 bytes per row instead of 4 bytes per entry of
 * row indices and sum every row from +0.0 in storage order, np.add.at
 * order): 2 on the column-panel path, 3 on the CSR tile kernel (plans
 * without long runs, unless tile / groups / warp_stream are configured or
 * spmv_plan_config.panels is 0).  The view serves products called with the
 * arrays the plan was created from. */
int spmv_coo_plan_path(const spmv_coo_plan* plan, int* warp_stream, int64_t* nwarps);
int spmv_coo_plan_groups(const spmv_coo_plan* plan, int* groups);

/* Fixed 1536-entry tiles (TMA bulk copies; 7 consumer groups over an 8-stage
 * ring, or one group when long runs exist), segmented without atomics: rows
 * of at most 32 entries are summed left to right by one thread starting
 * from +0.0 (bit-exact with np.add.at); longer runs are reduced in 256-entry
 * vla-32 units, cross-tile parts combined in tile order by a fix-up kernel. */
int spmv_coo(const spmv_coo_plan* plan, const uint32_t* row_indices,
             const uint32_t* col_indices, const void* values, const void* x,
             int64_t col_base, int64_t x_len, void* y, void* stream);

/* Requires the reference's `sorted` flag (kernels.py:119-120; checked by
 * the caller).  Per row: chunks of L entries, each tree-reduced, added once
 * into y: bit-exact with spmv_coo_vla.  outer_steps (may be NULL) receives
 * the reference's step count (kernels.py:138-140); non-NULL synchronises.
 * Runs over 256 entries take a two-phase path (step trees over all warps,
 * then an ordered fold per run) whose buffers the plan keeps (built on the
 * first call that needs them; not reentrant per plan). */
int spmv_coo_vla(spmv_coo_plan* plan, const uint32_t* row_indices,
                 const uint32_t* col_indices, const void* values,
                 const void* x, int64_t col_base, int64_t x_len, void* y,
                 int lanes, int64_t* outer_steps, void* stream);

/* ---- DIA (kernels.py:85-101 spmv_dia_plain, :174-210 spmv_dia_vla) ----- */
/* Rows [0, nrows) of the block `values` (row stride ndiags) are the global
 * rows [row_base, row_base + nrows); avail_rows >= nrows rows of the block
 * are readable (padding included).  Column bound checks use the global
 * ncols; x is the window starting at global column col_base.  Each row sums
 * its in-bounds diagonals in ascending offset order from +0.0, so the
 * result is bit-exact with spmv_dia_plain and spmv_dia_vla (any lanes). */
int spmv_dia(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags,
             int64_t avail_rows, const int32_t* offsets, const void* values,
             const void* x, int64_t row_base, int64_t col_base, int64_t x_len,
             void* y, void* stream);

/* spmv_dia with the DIA fields of a configuration (dia_kernel, dia_rows,
 * ctas_per_sm); NULL = auto, same as spmv_dia. */
int spmv_dia_ex(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags,
                int64_t avail_rows, const int32_t* offsets, const void* values,
                const void* x, int64_t row_base, int64_t col_base, int64_t x_len,
                void* y, const spmv_plan_config* cfg, void* stream);

/* spmv_dia with a gap: launch rows v >= y_split are slab rows v + y_gap
 * (their values, x reach and y), so a rank's two boundary blocks run as one
 * launch after the halo exchange.  nrows and avail_rows count launch rows
 * (avail_rows = slab rows available from `values` minus y_gap).  When
 * y_split falls on the kernel's row-tile boundary R (R = 256 rows for up to
 * 28 f64 / 56 f32 diagonals, fewer for wider rows) and y_gap rows are a
 * 16-byte multiple of the row bytes, both blocks run in one launch;
 * otherwise the call runs them as two spmv_dia launches (same result). */
int spmv_dia_gapped(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags,
                    int64_t avail_rows, const int32_t* offsets, const void* values,
                    const void* x, int64_t row_base, int64_t col_base, int64_t x_len,
                    void* y, int64_t y_split, int64_t y_gap, void* stream);

/* ---- conversions (convert.py) ------------------------------------------ */
/* convert.py:87-94: IRP from a sorted COO (copies AJ/AV too). */
int spmv_coo_to_csr(int dtype, int64_t nrows, int64_t nnz,
                    const uint32_t* row_indices, const uint32_t* col_indices,
                    const void* values, uint32_t* row_pointers_out,
                    uint32_t* col_indices_out, void* values_out, void* stream);

/* convert.py:97-110: row expansion; *sorted_out = 1 iff columns strictly
 * increase inside every row.  Synchronises. */
int spmv_csr_to_coo(int dtype, int64_t nrows, int64_t nnz,
                    const uint32_t* row_pointers, const uint32_t* col_indices,
                    const void* values, uint32_t* row_indices_out,
                    uint32_t* col_indices_out, void* values_out,
                    int* sorted_out, void* stream);

/* convert.py:113-144: two phases so the host can apply the DiaFillPolicy
 * before the block is allocated (convert.py:128-139). */
typedef struct spmv_dia_builder spmv_dia_builder;
int spmv_coo_to_dia_analyze(int64_t nrows, int64_t ncols, int64_t nnz,
                            const uint32_t* row_indices,
                            const uint32_t* col_indices, void* stream,
                            spmv_dia_builder** out, int64_t* ndiags_out);
int spmv_coo_to_dia_offsets(const spmv_dia_builder* b, int32_t* offsets_out,
                            void* stream);
/* values_out: (padded_rows, ndiags) row-major, fully written (zeros +
 * scatter). */
int spmv_coo_to_dia_fill(const spmv_dia_builder* b, int dtype,
                         int64_t padded_rows, const uint32_t* row_indices,
                         const uint32_t* col_indices, const void* values,
                         void* values_out, void* stream);
int spmv_dia_builder_destroy(spmv_dia_builder* b);

/* convert.py:147-177: in-bounds cells != 0 (NaN kept, -0.0 dropped), in
 * (row, col) order.  count synchronises; fill writes nnz_out triples. */
typedef struct spmv_dia_collect spmv_dia_collect;
int spmv_dia_to_coo_count(int dtype, int64_t nrows, int64_t ncols,
                          int64_t ndiags, const int32_t* offsets,
                          const void* values, void* stream,
                          spmv_dia_collect** out, int64_t* nnz_out);
int spmv_dia_to_coo_fill(const spmv_dia_collect* c, int dtype,
                         const int32_t* offsets, const void* values,
                         uint32_t* row_indices_out, uint32_t* col_indices_out,
                         void* values_out, void* stream);
int spmv_dia_collect_destroy(spmv_dia_collect* c);

/* convert.py:60-84: stable (row, col) sort; duplicate coordinates summed in
 * numpy's np.add.reduceat order (first element + pairwise sum of the rest,
 * numpy 2.3 pairwise_sum), zero sums kept.  One call: a stable radix sort on
 * the row with the storage index as payload, then each row's columns sorted
 * (warp bitonic sort for rows of <= 32 entries, a segmented sort above),
 * duplicates merged only when some (row, column) repeats.  The outputs have
 * capacity nnz; *nnz_out receives the merged count.  Synchronises. */
int spmv_sort_coo(int dtype, int64_t nrows, int64_t ncols, int64_t nnz,
                  const uint32_t* row_indices, const uint32_t* col_indices,
                  const void* values, uint32_t* row_indices_out,
                  uint32_t* col_indices_out, void* values_out,
                  int64_t* nnz_out, void* stream);

/* ---- generators (matrixio.py:170-210 gen_stencil27) -------------------- */
/* nnz = prod(3*n_d - 2) (1 for n_d = 1).  IndexOverflow when 27*n > 2^32-1
 * (matrixio.py:182-183). */
int spmv_stencil27_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t* nnz_out);
/* Rows [row_begin, row_end) of the global stencil operator; row_pointers_out
 * gets (row_end - row_begin + 1) entries rebased to start at 0. */
int spmv_stencil27_fill(int dtype, int64_t nx, int64_t ny, int64_t nz,
                        int64_t row_begin, int64_t row_end,
                        uint32_t* row_pointers_out, uint32_t* col_indices_out,
                        void* values_out, void* stream);

/* ---- row-partition helpers (hpcg.py:95-189) ---------------------------- */
/* Min and max column referenced by rows [0, nrows) of a CSR block
 * (min = UINT32_MAX, max = 0 when empty).  Synchronises. */
int spmv_csr_col_bounds(int64_t nrows, const uint32_t* row_pointers,
                        const uint32_t* col_indices, void* stream,
                        uint32_t* min_out, uint32_t* max_out);

/* Rows of a CSR slab that need no halo: every row in [*i_lo, *i_hi) reads
 * only columns in [col_lo, col_hi).  *i_lo = 1 + last row reading a column
 * below col_lo (0 if none); *i_hi = first row reading a column >= col_hi
 * (nrows if none).  Lets the interior rows run while the halo exchange is in
 * flight (hpcg.py:157-180 split into overlap-able parts).  Synchronises. */
int spmv_csr_halo_split(int64_t nrows, const uint32_t* row_pointers,
                        const uint32_t* col_indices, int64_t col_lo,
                        int64_t col_hi, void* stream, int64_t* i_lo,
                        int64_t* i_hi);

/* ---- CG vector kernels (hpcg.py:211-258) ------------------------------- */
/* Deterministic dot product: ws holds spmv_dot_workspace_entries() values;
 * the result lands in ws[entries-1] (device).  Fixed reduction tree, run to
 * run identical and independent of the SM count. */
int spmv_dot_workspace_entries(void);
int spmv_dot(int dtype, int64_t n, const void* a, const void* b, void* ws,
             void* stream);
/* x += alpha p; r -= alpha Ap (rounded products, no FMA, hpcg.py:243-246);
 * the new r.r lands in ws[entries-1] like spmv_dot. */
int spmv_cg_update(int dtype, int64_t n, double alpha, const void* p,
                   const void* ap, void* x, void* r, void* ws, void* stream);
/* p = r + beta p (hpcg.py:253). */
int spmv_cg_direction(int dtype, int64_t n, double beta, const void* r,
                      void* p, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPMV_B200_H */
