/*
 * dmath_b200 -- C ABI of the B200-native distributed fp32 GEMM path.
 *
 * Drop-in boundary for the reference's distributed-matrix/GEMM API
 * (arxiv 1604.01416 "dMath", code under /root/reference/proj/include/gridgemm).
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj/include/gridgemm/).  Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.
 *
 * All functions return a dm_status (0 = ok).  On error, dm_last_error()
 * returns the message of the failing call on this thread; the code maps 1:1
 * onto the reference's exception classes (common.hpp:22-78).
 */
#ifndef DMATH_B200_H_
#define DMATH_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMATH_B200_ABI_VERSION 2

/* ---- status codes: reference exception classes (common.hpp:22-78) ---- */
enum dm_status {
  DM_OK = 0,
  DM_ERR_USAGE = 1,       /* UsageError      common.hpp:28-32 */
  DM_ERR_CONFIG = 2,      /* ConfigError     common.hpp:34-38 */
  DM_ERR_SHAPE = 3,       /* ShapeError      common.hpp:40-44 */
  DM_ERR_PROTOCOL = 4,    /* ProtocolError   common.hpp:46-51 */
  DM_ERR_DEADLOCK = 5,    /* DeadlockError   common.hpp:53-57 */
  DM_ERR_INTEGRITY = 6,   /* IntegrityError  common.hpp:59-63 */
  DM_ERR_PLAN = 7,        /* PlanError       common.hpp:65-70 */
  DM_ERR_CACHE_MISS = 8,  /* CacheMissError  common.hpp:72-78 */
  DM_ERR_CUDA = 9,        /* device runtime failure (no reference equivalent) */
  DM_ERR_NCCL = 10,       /* NCCL failure (no reference equivalent) */
  DM_ERR_UNSUPPORTED = 11 /* reserved: an operation this build does not provide */
};

/* ---- enums mirroring the reference ---- */
enum dm_layout_kind { /* layout.hpp:69-75 */
  DM_ROW_BLOCKS_1D = 0,
  DM_COL_BLOCKS_1D = 1,
  DM_ROW_CYCLIC_1D = 2,
  DM_CHECKERBOARD_2D = 3,
  DM_CUSTOM = 4
};
enum dm_precision { DM_HALF16 = 0, DM_SINGLE32 = 1, DM_DOUBLE64 = 2 }; /* precision.hpp:14 */
enum dm_fill { DM_FILL_ZEROS = 0, DM_FILL_SEEDED = 1, DM_FILL_FROM_HOST = 2 }; /* runtime_types.hpp:68 */
/* Split-product scheme of the fp32 tensor-core GEMM (all fp32-accurate,
 * DESIGN.md section 4):
 *   DM_GEMM_MIXED  : hi*hi as tcgen05 kind::tf32 + the two cross terms as bf16
 *                    (kind::f16): 4 bf16-MMA slots per useful k16;
 *   DM_GEMM_TF32X3 : lo*hi + hi*lo + hi*hi, all kind::tf32 (north star's
 *                    3xTF32): 6 slots per k16;
 *   DM_GEMM_F16X2  : 3xTF32's numerics on fp16 operands -- per plane row a
 *                    power-of-two scale puts max|x| in [2^14, 2^15), then
 *                    x*2^e = h0 + h1 (fp16, 11 + 11 bits like tf32 hi / lo) and
 *                    h1*h0 + h0*h1 + h0*h0 as kind::f16: 3 slots per k16, 4 B of
 *                    planes per element;
 *   DM_GEMM_AUTO   : f16x2 (3xTF32's accuracy at 1.8x its speed), except for
 *                    latency-bound products -- below DM_F16X2_MIN_GFLOP
 *                    (default 64) GFLOP per worker / call -- which run 3xTF32
 *                    (one-pass split); Half16 operands run 3xTF32;
 *   DM_GEMM_DEFAULT: the DM_GEMM_MODE environment variable (0 = 3xTF32,
 *                    1 = mixed, 2 = auto, 3 = f16x2), else auto. */
enum dm_gemm_mode { DM_GEMM_DEFAULT = 0, DM_GEMM_MIXED = 1, DM_GEMM_TF32X3 = 2, DM_GEMM_AUTO = 3, DM_GEMM_F16X2 = 4 };
enum dm_mode {
  DM_MODE_LOCAL = 0, /* one process drives every worker (reference Session, session.hpp:64-76) */
  DM_MODE_SPMD = 1   /* one process per GPU; every rank makes the same calls (torchrun) */
};

/* LayoutSpec (layout.hpp:116-142): block grid + kind + worker count.
 * `custom` is the row-major n_block_rows x n_block_cols owner table (Custom only). */
typedef struct dm_layout {
  int32_t kind;
  int32_t worker_count;
  int64_t global_rows, global_cols;
  int64_t block_rows, block_cols;
  const int32_t* custom;
  int64_t custom_len;
} dm_layout;

/* Pool::Stats (pool.hpp:63-69), per worker device pool. */
typedef struct dm_pool_stats {
  uint64_t fresh_allocations;
  uint64_t reuses;
  uint64_t bytes_live;
  uint64_t bytes_pooled;
  uint64_t high_water;
} dm_pool_stats;

/* Data-movement and kernel counters of one worker (cumulative). */
typedef struct dm_worker_stats {
  uint64_t peer_bytes_read;   /* operand bytes pulled from other workers' blocks */
  uint64_t local_bytes_read;  /* operand bytes read from own owned/cached blocks */
  uint64_t gemm_launches;     /* tcgen05 GEMM kernel launches */
  uint64_t split_launches;    /* split/pull kernel launches */
  double gemm_flops;          /* algorithmic 2*m*n*k of those launches */
  double gemm_ms;             /* CUDA-event time of the GEMM launches (timing enabled) */
} dm_worker_stats;

/* MatrixDescriptor (layout.hpp:224-236). */
typedef struct dm_descriptor {
  uint64_t matrix_id;
  int32_t precision;
  int32_t replicated;
  uint64_t version;
  uint64_t replica_version;
  uint64_t seed;
  dm_layout layout; /* layout.custom points into session-owned storage */
} dm_descriptor;

/* One worker-to-worker block transfer (TransferRecord, transport.hpp:27-38):
 * `bytes` = payload read from src's block (a GEMM may read part of a block). */
typedef struct dm_transfer_record {
  uint64_t seq;
  int32_t src, dst;
  uint64_t matrix_id;
  int32_t row, col;
  uint64_t bytes;
  char op[32];
} dm_transfer_record;

typedef struct dm_session_config {
  int32_t worker_count;     /* P (Config::worker_count, session.hpp:56) */
  int32_t mode;             /* dm_mode */
  int32_t rank;             /* SPMD: this process's worker id */
  int32_t coherence_checks; /* Config::coherence_checks (session.hpp:61) */
  uint64_t root_seed;       /* Config::root_seed (session.hpp:59) */
  const int32_t* devices;   /* LOCAL: device of each worker (NULL = w % device_count) */
  const void* nccl_id;      /* SPMD: 128-byte ncclUniqueId from rank 0 (dm_nccl_unique_id) */
  int32_t gemm_mode;        /* dm_gemm_mode of every fp32/fp16 GEMM of the session */
} dm_session_config;

typedef struct dm_session dm_session;
typedef uint64_t dm_matrix_id;

/* ---- diagnostics ---- */
const char* dm_last_error(void);
/* CacheMissError::missing_coords of the last failure: fills up to cap (row,col)
 * pairs into coords[2*i], returns the total count. */
int dm_last_error_missing(int32_t* coords, int cap);
int dm_abi_version(void);

/* ---- host-only geometry (no GPU needed) ---- */
/* detail::checkerboard_dims (layout.hpp:100-105) */
int dm_checkerboard_dims(int workers, int* pr, int* pc);
/* LayoutSpec::owner (layout.hpp:122-139) */
int dm_layout_owner(const dm_layout* layout, int row, int col, int* owner);
/* BlockGrid::n_block_rows/cols (layout.hpp:34-40), clamped flag (make_grid, layout.hpp:49-59) */
int dm_layout_grid(const dm_layout* layout, int* n_block_rows, int* n_block_cols, int* clamped);
/* block_extent (layout.hpp:62-67) */
int dm_block_extent(const dm_layout* layout, int row, int col, int64_t* rows, int64_t* cols);
/* layout_to_string (layout.hpp:174-187); returns needed length incl. NUL */
int dm_layout_to_string(const dm_layout* layout, char* buf, int cap);
/* Pool::size_class (pool.hpp:121-125) */
uint64_t dm_pool_size_class(uint64_t bytes);
/* GEMM data-movement plan of worker `w` for general_gemm on these layouts:
 * counts the distinct peer blocks w must read (GeneralGemmExec::add_needed,
 * ops.hpp:503-524) and their bytes.  Pure host logic. */
int dm_plan_general_gemm(const dm_layout* a, int trans_a, const dm_layout* b, int trans_b,
                         const dm_layout* c, int worker, int64_t* peer_blocks,
                         int64_t* peer_bytes);
/* K panels of a presplit (owner-split) GEMM over K with A's / B's K-block
 * widths a_kblock / b_kblock and the widest panel `max_width`
 * (DM_PRESPLIT_PANEL): panel starts then K in out[0..*n-1] (at most cap
 * entries).  Pure host logic (before a worker's own lead-panel cut). */
int dm_presplit_panels(int64_t k, int64_t a_kblock, int64_t b_kblock, int64_t max_width, int64_t* out,
                       int cap, int* n);

/* ---- session (Session, session.hpp:53-485) ---- */
/* Session::Session (session.hpp:64-76).  SPMD: collective over all ranks. */
int dm_session_create(const dm_session_config* cfg, dm_session** out);
/* Session::~Session / shutdown (session.hpp:467-481). Idempotent. */
int dm_session_destroy(dm_session* s);
int dm_session_shutdown(dm_session* s);
int dm_nccl_unique_id(void* out128);

/* create_matrix (session.hpp:129-150); host used for DM_FILL_FROM_HOST
 * (row-major global_rows x global_cols, elements of `precision`). */
int dm_create_matrix(dm_session* s, const dm_layout* layout, int precision, int fill,
                     const void* host, dm_matrix_id* out);
/* destroy_matrix (session.hpp:152-160) */
int dm_destroy_matrix(dm_session* s, dm_matrix_id id);
/* scatter (session.hpp:164-175): host row-major rows x cols, bit-exact. */
int dm_scatter(dm_session* s, dm_matrix_id id, const void* host, int64_t rows, int64_t cols);
/* gather (session.hpp:179-201): owned blocks only, bit-exact.  root >= 0:
 * the full matrix lands in `host` of worker `root`'s process (SPMD) --
 * LOCAL sessions always fill the whole matrix; root = -1 (SPMD): every rank
 * writes only the blocks it owns into its own `host`. */
int dm_gather(dm_session* s, dm_matrix_id id, void* host, int64_t rows, int64_t cols, int root);
/* update_block (session.hpp:203-222): one block from host data of the
 * matrix's precision (rows x cols = the block extent); version += 1. */
int dm_update_block(dm_session* s, dm_matrix_id id, int row, int col, const void* host,
                    int64_t rows, int64_t cols);
/* replicate (session.hpp:266-274): every worker keeps version-tagged copies
 * of all blocks it does not own (ReplicateExec, ops.hpp:660-702). */
int dm_replicate(dm_session* s, dm_matrix_id id, int enable);
/* replica_read (session.hpp:276-297): lazy resync of stale replicas, then the
 * full matrix assembled from worker `reader` (its process fills `host`). */
int dm_replica_read(dm_session* s, dm_matrix_id id, int reader, void* host, int64_t rows,
                    int64_t cols);
/* reshape (session.hpp:299-317): new matrix, same row-major element order,
 * any layout/precision; narrowing happens before the link (ops.hpp:772-944). */
int dm_reshape(dm_session* s, dm_matrix_id src, const dm_layout* layout, int precision,
               dm_matrix_id* out);
/* add_row_col_sum (session.hpp:321-348): axis 0 = row sums (global_rows x 1),
 * 1 = column sums; deterministic != 0 folds partials in worker order. */
int dm_add_row_col_sum(dm_session* s, dm_matrix_id id, int axis, int deterministic,
                       dm_matrix_id* out);
/* checkpoint / restore (session.hpp:395-465), "DMTH" v1 file format of
 * checkpoint.hpp:1-12 (interchangeable with the reference's files). */
int dm_checkpoint(dm_session* s, const char* path);
int dm_restore(const char* path, const dm_session_config* cfg, dm_session** out);

/* general_gemm (session.hpp:244-250): C <- alpha op(A) op(B) + beta C.
 * Single32 / Half16: tcgen05, within relFro 1e-5 of the reference;
 * Double64: bit-exact with gemm_typed<double> (kernels.hpp:48-75). */
int dm_general_gemm(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b, double beta,
                    dm_matrix_id c, int trans_a, int trans_b);
/* cyclic_gemm (session.hpp:226-234): ring-plan preconditions (ops.hpp:84-169) */
int dm_cyclic_gemm(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b, double beta,
                   dm_matrix_id c, int trans_a, int trans_b, int cache_a);
/* broadcast_gemm_reference (session.hpp:236-242) */
int dm_broadcast_gemm_reference(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b,
                                double beta, dm_matrix_id c, int trans_a, int trans_b);
/* cached_backward_gemm (session.hpp:254-264): dX <- W dY, zero transfers */
int dm_cached_backward_gemm(dm_session* s, dm_matrix_id w, dm_matrix_id dy, dm_matrix_id dx);

/* ---- introspection ---- */
int dm_worker_count(dm_session* s, int* out);
int dm_local_workers(dm_session* s, int32_t* ids, int cap); /* returns count */
int dm_descriptor_get(dm_session* s, dm_matrix_id id, dm_descriptor* out); /* session.hpp:93-97 */
int dm_pool_stats_get(dm_session* s, int worker, dm_pool_stats* out);     /* session.hpp:102 */
int dm_pool_trim(dm_session* s, int worker, uint64_t* freed);             /* pool.hpp:110-115 */
int dm_worker_stats_get(dm_session* s, int worker, dm_worker_stats* out);
int dm_worker_stats_reset(dm_session* s);
/* Record CUDA events around every GEMM launch (fills gemm_ms). */
int dm_set_gemm_timing(dm_session* s, int enable);
int dm_worker_seed(dm_session* s, int worker, uint64_t* out); /* session.hpp:103 */
/* The session's resolved split-product scheme: DM_GEMM_MIXED, DM_GEMM_TF32X3 or DM_GEMM_AUTO. */
int dm_session_gemm_mode(dm_session* s, int* out);
/* Host-only: the scheme (DM_GEMM_MIXED, DM_GEMM_TF32X3 or DM_GEMM_F16X2) a
 * product over `k` with `work` = 2 m n k flops per worker (< 0: unknown) runs
 * in under `gemm_mode` (DM_GEMM_DEFAULT reads DM_GEMM_MODE; auto's rule). */
int dm_split_mode_for(int gemm_mode, int64_t k, double work, int* out);
/* trace() (session.hpp:94; TraceLog, transport.hpp:56-71): the block transfers
 * this process's workers pulled, oldest first; fills up to cap records and
 * returns the total count (negative status on error). */
int dm_transfer_log(dm_session* s, dm_transfer_record* out, int cap);
/* root_seed (session.hpp:92): current root (after seed_workers / restore). */
int dm_root_seed(dm_session* s, uint64_t* out);
/* seed_workers (session.hpp:115-125): new root seed for worker seeds and for
 * matrices created afterwards; seeds[w] = mix64(root, w) for w < cap. */
int dm_seed_workers(dm_session* s, uint64_t root, uint64_t* seeds, int cap);
int dm_descriptor_digest(dm_session* s, uint64_t* master, uint64_t* workers, int cap);
/* device pointer of an owned block (for tests / zero-copy interop) */
int dm_block_device_ptr(dm_session* s, dm_matrix_id id, int row, int col, void** ptr,
                        int* device);
int dm_barrier(dm_session* s);
/* Asynchronous command mode (on != 0): dm_scatter / dm_gather / dm_general_gemm
 * enqueue stream-ordered work on copy-engine / compute / pull streams and
 * return; per-matrix read/write events (and device-side NCCL barriers across
 * ranks) keep them ordered, so H2D, tensor-core and D2H work overlap.  Host
 * buffers passed to scatter/gather must stay valid and unmodified until
 * dm_barrier() or dm_set_async(s, 0); other commands drain first and run
 * synchronously.  The reference's calls are synchronous (session.hpp:585-605);
 * this mode is the B200 extension of the same command stream. */
int dm_set_async(dm_session* s, int on);
/* Device-time markers on worker `worker`'s GEMM stream (bench timing):
 * record CUDA event `slot` (0..15); elapsed ms between two recorded slots. */
int dm_marker_record(dm_session* s, int worker, int slot);
int dm_marker_elapsed(dm_session* s, int worker, int slot_a, int slot_b, float* ms);

/* ---- the per-worker BLAS seam: local_gemm (kernels.hpp:81-89) on device
 * memory.  op(A) is m x k (A stored k x m when trans_a), op(B) is k x n (B
 * stored n x k when trans_b), row pitches in elements.  Stream-ordered on
 * `stream` (cudaStream_t, NULL = legacy default): the call only enqueues work
 * and returns; its scratch (split planes) comes from a per-device pool and is
 * recycled once an event after its kernels fired, so calls on different
 * streams may run concurrently.  Inside a CUDA-graph capture use
 * dm_local_gemm_f32_ws (the graph must own its scratch); these two return
 * DM_ERR_USAGE there. ---- */
int dm_local_gemm_f32(double alpha, const float* a, int64_t lda, int trans_a, const float* b,
                      int64_t ldb, int trans_b, double beta, float* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, void* stream);
/* Same, choosing the tile shape (cta_group 0 = auto, 1 = 128x128 tiles, 2 =
 * 256x256 CTA-pair tiles) and the split-product scheme (dm_gemm_mode). */
int dm_local_gemm_f32_ex(double alpha, const float* a, int64_t lda, int trans_a, const float* b,
                         int64_t ldb, int trans_b, double beta, float* c, int64_t ldc, int64_t m,
                         int64_t n, int64_t k, int cta_group, int gemm_mode, void* stream);
/* Caller-owned scratch: bytes of workspace a dm_local_gemm_f32_ws call with
 * these arguments needs on the current device (0 when m, n or k is 0). */
int dm_local_gemm_f32_workspace_size(int64_t m, int64_t n, int64_t k, int cta_group, int gemm_mode,
                                     size_t* bytes);
/* local_gemm with a caller workspace (256-byte aligned, >= the size above):
 * no allocation, no host synchronisation, capturable in a CUDA graph. */
int dm_local_gemm_f32_ws(double alpha, const float* a, int64_t lda, int trans_a, const float* b,
                         int64_t ldb, int trans_b, double beta, float* c, int64_t ldc, int64_t m,
                         int64_t n, int64_t k, int cta_group, int gemm_mode, void* workspace,
                         size_t workspace_bytes, void* stream);
/* WorkerContext::fill_seeded (runtime_types.hpp:208-218) for one block. */
int dm_fill_seeded_f32(float* dst, int64_t count, uint64_t matrix_seed, int block_row,
                       int block_col, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DMATH_B200_H_ */
