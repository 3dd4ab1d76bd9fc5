/*
 * dbf_b200.h -- C ABI of the B200-native Double Binary Factorization (DBF) forward path.
 *
 * The reference (arxiv 2505.11076, package `dbf` 0.1.0 under /root/reference/pkg) exposes the
 * hot path as plain Python functions with no FFI layer:
 *
 *   pack(dense) -> SignMatrix                pkg/src/dbf/bitcore.py:72-85
 *   unpack(s)   -> ndarray                   pkg/src/dbf/bitcore.py:88-91
 *   sign_matvec(s, x) -> ndarray             pkg/src/dbf/kernel.py:24-45
 *   forward(X, layer) -> ndarray             pkg/src/dbf/kernel.py:48-62
 *
 * Each entry point below replaces one of them (cited per function).  The Python package
 * `paper_2505_11076_b200` binds this ABI through ctypes and re-exposes the reference
 * signatures and error messages; see INTEGRATION.md for the binding a maintainer would add.
 *
 * Conventions (all functions):
 *   - plain C types only; pointers are DEVICE pointers unless stated otherwise;
 *   - every call is asynchronous on the caller's `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream) and never synchronises the device;
 *   - no hidden device allocation: scratch memory is a caller-provided workspace whose size
 *     is returned by the matching *_workspace_bytes() query;
 *   - return value is a dbf_status (0 = DBF_OK); nothing throws across the ABI;
 *   - sign bit semantics follow the reference exactly: bit value 1 <=> +1, 0 <=> -1
 *     (bitcore.py:7-9), columns LSB-first inside each byte/word.
 *
 * Device layouts:
 *   canonical  : uint32 words, row-major, word j of a row holds columns 32j..32j+31 (bit i <->
 *                column 32j+i).  This is the reference's uint8 row bytes viewed little-endian as
 *                uint32, with the row pitch padded to `dbf_canonical_pitch_words(cols)` words
 *                (a multiple of 4 words = 16 bytes) and every padding bit zero.
 *   tiled      : the decode engine's operand layout.  Rows are grouped in blocks of 16, columns
 *                in chunks of 256; one (row block, chunk) is 512 contiguous bytes = 32 lanes x
 *                4 words, ordered so that one 128-bit load per lane yields the A fragments of
 *                eight int8 m16n8k32 tensor-core MMAs after a single AND per register.
 */
#ifndef DBF_B200_H
#define DBF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBF_ABI_VERSION 1

typedef enum {
  DBF_OK = 0,
  DBF_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative/zero size, bad dtype              */
  DBF_ERR_SHAPE = 2,            /* dimension mismatch between operands                       */
  DBF_ERR_WORKSPACE = 3,        /* workspace too small                                       */
  DBF_ERR_CUDA = 4,             /* a CUDA runtime call failed (see dbf_last_cuda_error)      */
  DBF_ERR_UNSUPPORTED = 5       /* configuration not supported by this build                 */
} dbf_status;

typedef enum {
  DBF_F16 = 0,
  DBF_F32 = 1,
  DBF_F64 = 2,
  DBF_BF16 = 3
} dbf_dtype;

/* ---- library metadata ------------------------------------------------------------------ */
int dbf_abi_version(void);
const char* dbf_status_string(int status);
/* cudaError_t of the last failing CUDA call made by this library on the calling thread. */
int dbf_last_cuda_error(void);
const char* dbf_last_cuda_error_string(void);

/* ---- layout queries (host-only arithmetic, safe without a GPU) ------------------------- */
/* bitcore.row_bytes (bitcore.py:67-69): bytes of one reference-packed row. */
int64_t dbf_row_bytes(int64_t cols);
/* words per row of the canonical device layout (multiple of 4). */
int64_t dbf_canonical_pitch_words(int64_t cols);
/* bytes of the tiled decode layout of a rows x cols sign matrix. */
int64_t dbf_tiled_bytes(int64_t rows, int64_t cols);

/* ---- bitcore: pack / unpack (bitcore.py:72-91) ------------------------------------------ */
/*
 * dbf_pack_signs -- replaces bitcore.pack (bitcore.py:72-85).
 * dense: rows x cols values of `dtype` (F16/F32/F64/BF16) with leading dimension `ld`
 * (elements).  Writes canonical words (pitch `word_pitch` >= dbf_canonical_pitch_words(cols)).
 * Validation matches the reference: every entry must be exactly +1 or -1 (|v| == 1; NaN and 0
 * are rejected).  *d_first_bad (a device int64) receives the row-major linear index r*cols+c of
 * the FIRST offending entry, or -1 when all entries are valid.  The caller reads it back and
 * raises ValueError("entry at (r, c) is v, expected -1 or +1") like bitcore.py:81-82.
 */
int dbf_pack_signs(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t ld,
                   uint32_t* words, int64_t word_pitch, int64_t* d_first_bad, void* stream);

/* dbf_pack_sign_of -- pack(np.where(Z >= 0, 1, -1)) of svid.svid (svid.py:99-103): bit = (v >= 0),
 * canonical words, no +-1 validation (the caller rejects non-finite input like as_matrix). */
int dbf_pack_sign_of(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t ld,
                     uint32_t* words, int64_t word_pitch, void* stream);

/* dbf_unpack_signs -- replaces bitcore.unpack (bitcore.py:88-91): canonical words -> +-1. */
int dbf_unpack_signs(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                     void* dense, int dtype, int64_t ld, void* stream);

/*
 * dbf_repack_u8 -- upload path of SignMatrix.bits (bitcore.py:40-64): reference row bytes
 * (rows x dbf_row_bytes(cols), contiguous, device) -> canonical words.  Padding bits of the last
 * byte are cleared, so flipped padding bits never contribute (test_kernel.py:35-45).
 */
int dbf_repack_u8(const uint8_t* bytes, int64_t rows, int64_t cols, uint32_t* words,
                  int64_t word_pitch, void* stream);

/* dbf_words_to_u8 -- canonical words -> reference row bytes (rows x dbf_row_bytes(cols)). */
int dbf_words_to_u8(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                    uint8_t* bytes, void* stream);

/* dbf_transpose_signs -- canonical words of S (rows x cols) -> canonical words of S^T (cols x rows,
 * pitch out_pitch >= dbf_canonical_pitch_words(rows)); padding bits zero.  Feeds the transposed
 * sign products of the staged gradients (budget.channel_scores, budget.py:145-173;
 * factorize._staged_loss_grads / refine_scales, factorize.py:310-370). */
int dbf_transpose_signs(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                        uint32_t* out, int64_t out_pitch, void* stream);

/* dbf_sign_gemm_f64 -- out[i, r] = sum_c S[r, c] * x[i, c] in float64 on CUDA cores (canonical
 * words; x: batch x cols, stride ldx; out: batch x rows, stride ldo).  The float64 sign products of
 * the staged gradients (budget.py:158-168, factorize.py:310-326), where the reference's tests
 * compare exact zeros and equalities. */
int dbf_sign_gemm_f64(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                      const double* x, int64_t ldx, int64_t batch, double* out, int64_t ldo, void* stream);

/* dbf_tile_signs -- canonical words -> tiled decode layout (dbf_tiled_bytes(rows, cols)). */
int dbf_tile_signs(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                   void* tiled, void* stream);

/* ---- kernel: sign_matvec / forward (kernel.py:24-62) ------------------------------------ */
/*
 * Workspace for dbf_sign_matvec / dbf_forward.  batch = number of input rows of X.
 */
size_t dbf_forward_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch);

/*
 * dbf_sign_matvec -- replaces kernel.sign_matvec (kernel.py:24-45), batched:
 *   Y[i, r] = sum_c S[r, c] * X[i, c]      for i < batch, r < rows
 * S is given in the tiled layout.  X: batch x cols of x_dtype (F16/F32/F64), row stride ldx
 * elements.  Y: batch x rows of y_dtype (F16/F32/F64), row stride ldy.  The input row is
 * quantized once to a 22-bit fixed-point grid relative to its max |value| and the sum is
 * accumulated exactly in integers on the tensor cores, so the result is bitwise reproducible
 * (kernel.py:26-28).
 */
int dbf_sign_matvec(const void* S_tiled, int64_t rows, int64_t cols, const void* X, int x_dtype,
                    int64_t batch, int64_t ldx, void* Y, int y_dtype, int64_t ldy, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * dbf_forward -- replaces kernel.forward (kernel.py:48-62):
 *   Y[i] = a * (A . (mid * (B . (X[i] * b))))
 * A: n x k, B: k x m, both tiled.  a (n), mid (k), b (m) are scale vectors of scale_dtype
 * (F16, F32 or F64).  X: batch x m (x_dtype F16/F32/F64, stride ldx); Y: batch x n (y_dtype, stride
 * ldy).  The intermediate t = mid * (B . (b * x)) lives in the workspace as fp32.
 */
int dbf_forward(const void* A_tiled, const void* B_tiled, const void* a, const void* mid,
                const void* b, int scale_dtype, int64_t n, int64_t k, int64_t m, const void* X,
                int x_dtype, int64_t batch, int64_t ldx, void* Y, int y_dtype, int64_t ldy,
                void* workspace, size_t workspace_bytes, void* stream);

/*
 * dbf_forward_partial -- one middle-dimension (k) shard of dbf_forward for multi-GPU
 * tensor parallelism: the shard owns rows [k0,k1) of B, columns [k0,k1) of A
 * (passed as their own tiled n x (k1-k0) matrix) and mid[k0:k1].  Writes the fp32 partial
 *   P[i] = A_shard . (mid_shard * (B_shard . (X[i] * b)))      (no `a` scaling)
 * so that y = a * sum_over_shards(P) after an all-reduce (dbf_finalize_partial).
 */
int dbf_forward_partial(const void* A_shard_tiled, const void* B_shard_tiled,
                        const void* mid_shard, const void* b, int scale_dtype, int64_t n,
                        int64_t k_shard, int64_t m, const void* X, int x_dtype, int64_t batch,
                        int64_t ldx, float* P, void* workspace, size_t workspace_bytes,
                        void* stream);

/* y[i, r] = a[r] * P[i, r]  (P fp32 batch x n, contiguous) -> y_dtype with stride ldy. */
int dbf_finalize_partial(const float* P, const void* a, int scale_dtype, int64_t n, int64_t batch,
                         void* Y, int y_dtype, int64_t ldy, void* stream);

/*
 * dbf_forward_allreduce -- the k-sharded layer with its all-reduce fused into GEMV2 (SURVEY §8e,
 * step 2; replaces dbf_forward_partial + an NCCL all-reduce + dbf_finalize_partial, i.e. the
 * reference's kernel.forward, kernel.py:48-62, computed across `world` GPUs).  Every rank calls
 * it with the same n, batch and epoch.  GEMV2's epilogue stores each fp32 partial row block
 * straight into slot `rank` of every peer's receive buffer (NVLink P2P stores through mapped peer
 * addresses), then releases it with a per-(rank, row block) flag = epoch; each row block is then
 * combined on every rank as soon as all ranks have released it:
 *   Y[i, r] = a[r] * sum_{g = 0..world-1} P_g[i, r]   (rank order -> identical bits on all ranks)
 * peer_recv / peer_flags: DEVICE arrays of `world` device addresses (uint64) of every rank's
 * receive buffer (dbf_allreduce_recv_bytes) and flag array (dbf_allreduce_flag_bytes, zeroed
 * once before the first call), e.g. from torch symmetric memory.  epoch_counter: a LOCAL device
 * u32, zeroed with the flags; each call advances it on the device (so a captured CUDA graph
 * replays correctly) and uses the new value as its epoch: receive buffers alternate by epoch
 * parity and flags compare >= epoch, so nothing is cleared between calls.  batch <= 16.  A rank
 * that waits more than 20 s for a peer traps.
 */
size_t dbf_allreduce_recv_bytes(int64_t n, int64_t batch, int world);
size_t dbf_allreduce_flag_bytes(int64_t n, int world);
int dbf_forward_allreduce(const void* A_shard_tiled, const void* B_shard_tiled, const void* a,
                          const void* mid_shard, const void* b, int scale_dtype, int64_t n,
                          int64_t k_shard, int64_t m, const void* X, int x_dtype, int64_t batch,
                          int64_t ldx, void* Y, int y_dtype, int64_t ldy, const uint64_t* peer_recv,
                          const uint64_t* peer_flags, int world, int rank, uint32_t* epoch_counter,
                          void* workspace, size_t workspace_bytes, void* stream);

/*
 * Ablation kernel (north_star wording): the classic CUDA-core decode that XORs the fp16 sign
 * bit of x with the packed sign and accumulates with HADD2.  Same semantics as
 * dbf_sign_matvec for batch 1 but reads the canonical layout; kept only to measure against the
 * tensor-core path.
 */
int dbf_sign_matvec_xor(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                        const void* x, int x_dtype, float* y, void* stream);

/* ---- decode engine: a whole chain of DBF layers in ONE persistent kernel ---------------- */
/*
 * A program is a list of SEGMENTS (one sign GEMV each: y = oscale * (S . (iscale * v))) over
 * VECTORS, each holding `batch` tokens (1..4; every tensor-core MMA serves all of them: B columns
 * 2*token + digit plane).  Vector kind 0 = plain (dtype `dtype`, batch x len contiguous, ready when
 * the kernel starts, e.g. the token input); kind 1 = LL ("low-latency": uint32 words {fp16 value (low 16 bits), 16-bit epoch},
 * produced inside the kernel by another segment and consumed by polling the words themselves;
 * the buffer is padded to a multiple of 256 words).  Every segment's work is split into UNITS of
 * 16 rows; each CTA executes a list of RUNS -- up to dbf_engine_run_limits() consecutive units of
 * one segment, (segment, first row block, unit count) -- in order (cta_offsets[c] ..
 * cta_offsets[c+1]); dependencies are respected by construction (a run only reads vectors
 * written by runs of earlier stages).  One forward of a DBF layer is two segments: B with
 * iscale=b, oscale=mid -> t (LL), then A with oscale=a -> y.
 * Each CTA streams its runs' packed signs with cp.async.bulk into a shared-memory ring (one
 * producer warp) while 16 compute warps each own a set of 256-column chunks of the run's input:
 * a chunk is quantized (warp-local, relative to the chunk's max) as soon as its LL words carry
 * this launch's epoch and is multiplied on the int8 tensor cores against every unit of the run.
 * Outputs are fp16 (rounded once per layer stage); sums are exact integers per chunk, scaled and
 * accumulated in a fixed order, so results are bitwise reproducible run to run.
 */
typedef struct {
  const void* tiled;    /* tiled sign matrix (dbf_tile_signs) */
  int32_t rows, cols;   /* logical shape */
  int32_t in_vec;       /* input vector index */
  int32_t out_vec;      /* output LL vector index or -1 */
  const void* iscale;   /* per-column input scale or NULL */
  const void* oscale;   /* per-row output scale or NULL */
  int32_t scale_dtype;  /* F16 / F32 */
  int32_t out_dtype;    /* LL values are always rounded through fp16; out_plain is fp16 (F16) or the
                           unrounded fp32 value (F32) */
  void* out_plain;      /* optional plain output (out_dtype), NULL if unused */
} dbf_engine_segment;

typedef struct {
  void* data;           /* plain: batch x len values of `dtype`; LL: batch x (len padded to 256) uint32 words */
  int32_t len;
  int32_t kind;         /* 0 plain, 1 LL */
  int32_t dtype;        /* plain dtype (F16/F32) */
  int32_t producers;    /* LL: number of 16-row units that write it (filled by the builder) */
} dbf_engine_vector;

/* One RUN as the kernel consumes it: everything resolved on the host (no dependent metadata
 * loads on the device critical path).  Built by dbf_engine_build_runs. */
typedef struct {
  const void* tiled;        /* 0   first byte of the run's packed signs (row block rb)       */
  const void* x;            /* 8   input vector data                                          */
  const void* iscale;       /* 16  per-column input scale or NULL                             */
  const void* oscale;       /* 24  per-row output scale or NULL                               */
  void* out_plain;          /* 32  optional plain output                                      */
  void* ll_out;             /* 40  output LL vector data or NULL                              */
  uint32_t* ready_in;       /* 48  ready counter of the input vector (NULL for plain input)   */
  uint32_t* ready_out;      /* 56  ready counter of the output vector or NULL                 */
  int32_t rows, cols;       /* 64  segment shape                                              */
  int32_t rb, nunits;       /* 72  first row block, number of 16-row units                   */
  int32_t seg;              /* 80  segment index (the input is re-quantized when it changes)  */
  int32_t in_kind;          /* 84  0 plain, 1 LL                                              */
  int32_t in_dtype;         /* 88  plain input dtype                                          */
  int32_t scale_dtype;      /* 92                                                             */
  int32_t out_dtype;        /* 96                                                             */
  int32_t in_vec, out_vec;  /* 100 vector indices (LL epochs)                                 */
  uint32_t in_producers;    /* 108 units producing the input vector (ready target per run)    */
  int32_t pad[4];           /* 112 -> 128 bytes                                               */
} dbf_engine_run;

typedef struct {
  const dbf_engine_run* runs;         /* device array of run records, per CTA in order         */
  const int32_t* cta_offsets;         /* device array, grid + 1 entries (indices into runs)     */
  uint32_t* run_counter;              /* device uint32[4], zeroed once: [0] epoch base =
                                         (launches * nvectors) mod 65535 (the last CTA of a
                                         launch advances it; nvectors % 65535 != 0), [1] CTAs
                                         done, [2] sticky status bits: 1 = an input chunk held
                                         inf/NaN (the outputs it feeds are NaN), 2 = a value
                                         published in fp16 overflowed (|v| > 65504); the host
                                         reads and clears them, [3] reserved                    */
  int64_t* trace;                     /* optional: 4 x int64 %globaltimer stamps per run / NULL */
  int32_t nvectors;
  int32_t grid;                       /* CTAs (<= number of SMs; one per SM)                    */
  int32_t max_cols;                   /* largest segment `cols` (sizes shared memory)          */
  int32_t batch;                      /* tokens per step, 1..4 (vectors hold batch rows each)   */
  /* per-launch I/O (NULL = as built): x_override replaces the data of vector 0 (a plain input,
   * batch x len contiguous) and y_override the out_plain pointer of every segment that has one,
   * so one program serves calls on different input / output buffers without rebuilding runs */
  const void* x_override;
  void* y_override;
  /* batches of 2-4 tokens on inputs wider than the shared-memory store: a device buffer of
   * grid x qscratch_cta_bytes (dbf_engine_qscratch_bytes) where each CTA keeps its quantized
   * input chunks for the stage's later runs; NULL = re-quantize per run */
  void* qscratch;
  int64_t qscratch_cta_bytes;
  /* k-sharded layers: one-shot all-reduce fused into the program's last stage, the
   * engine counterpart of dbf_forward_allreduce (ar_world == 0: off).  Every segment with a plain
   * output pushes its unscaled fp32 rows into slot ar_rank of every peer's receive buffer
   * ([2][ar_world][ar_bt][rows] fp32, dbf_allreduce_recv_bytes), raises its row blocks in every
   * peer's flag array (group 0 of [16][ar_world][nrb] u32, dbf_allreduce_flag_bytes) after one
   * system-scope fence, waits for every rank's flags of those row blocks and writes
   * y[t, r] = ar_a[r] * sum over ranks in rank order (fp64, rounded once to fp32) to the plain
   * output (y_override or out_plain) as dtype ar_ydt, row stride ar_ldy.  The call's epoch is
   * *ar_epoch + 1 (the counter dbf_forward_allreduce also uses; the launch's last CTA advances
   * it), so calls of both paths may share one set of buffers. */
  const uint64_t* ar_recv;            /* device array [ar_world] of receive-buffer addresses    */
  const uint64_t* ar_flags;           /* device array [ar_world] of flag-array addresses        */
  uint32_t* ar_epoch;                 /* device call counter                                    */
  const void* ar_a;                   /* output scale a (n), dtype ar_sdt                       */
  int32_t ar_world, ar_rank, ar_bt, ar_sdt;
  int32_t ar_ydt, ar_pad;
  int64_t ar_ldy;
} dbf_engine_program;

/*
 * Host-only: resolve (segments, vectors, runs) -- HOST arrays, runs = 3 x int32 (segment, first
 * row block, units) per run -- into `nruns` run records written to the HOST buffer `out`.
 * `ready` is the DEVICE base address of the nvectors ready counters (zero-initialized).
 */
int dbf_engine_build_runs(const dbf_engine_segment* segments, int32_t nsegments,
                          const dbf_engine_vector* vectors, int32_t nvectors, const int32_t* runs,
                          int32_t nruns, int32_t batch, uint32_t* ready, dbf_engine_run* out);

/* Largest run the engine accepts at this batch: units per run and packed-sign bytes per run. */
int dbf_engine_run_limits(int32_t batch, int32_t* max_units, int64_t* max_run_bytes);
/* The same for a program whose widest segment has max_cols columns (at batch 1 the quantized-input
 * store grows with max_cols and the sign ring shrinks accordingly). */
int dbf_engine_run_limits_cols(int32_t max_cols, int32_t batch, int32_t* max_units, int64_t* max_run_bytes);
/* Per-CTA quantized-input scratch a program needs at this batch (0: none). */
size_t dbf_engine_qscratch_bytes(int32_t max_cols, int32_t batch);
/* Dynamic shared memory the engine needs for max_cols at this batch (1..4); DBF_ERR_UNSUPPORTED if
 * it cannot fit. */
int dbf_engine_smem_bytes(int32_t max_cols, int32_t batch, size_t* bytes);
/* Resident engine CTAs per SM and registers per thread for max_cols (diagnostics). */
int dbf_engine_occupancy(int32_t max_cols, int32_t* blocks_per_sm, int32_t* regs_per_thread);
/* Launch one run of the program (cooperative: all CTAs co-resident; one kernel). */
int dbf_engine_launch(const dbf_engine_program* program, void* stream);

/* ---- batched decode: 2-32 tokens, one pass over the weights -------------------------------- */
/*
 * dbf_forward (kernel.py:48-62) for a small token batch (batch <= 32): per stage, every extracted
 * sign fragment feeds one int8 IMMA per group of 4 tokens, so each sign matrix is read ONCE for
 * all tokens (the decode engine carries 4 tokens per launch).  Numerics are the engine's: each
 * (token, 256-column chunk) is quantized to a 13-bit grid relative to its chunk max (two balanced
 * int8 digit planes), chunk sums are exact integers, accumulation and the intermediate t are
 * fp32 (DESIGN.md §5 tolerance).  K is split over CTAs; split partials are summed in split order
 * (deterministic).  A non-finite input chunk makes the outputs it feeds NaN; `status` (optional,
 * device) gets bit 1 for a non-finite output and bit 2 for a finite value beyond the fp16 range.
 * Layouts: A / B tiled (dbf_tile_signs), X batch x m (stride ldx), Y batch x n (stride ldy).
 */
size_t dbf_forward_batched_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch);
int dbf_forward_batched(const void* A_tiled, const void* B_tiled, const void* a, const void* mid,
                        const void* b, int scale_dtype, int64_t n, int64_t k, int64_t m,
                        const void* X, int x_dtype, int64_t batch, int64_t ldx, void* Y,
                        int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes,
                        unsigned* status, void* stream);
/* The same, split for layer chains (DecodePlan.use_batched): a layer's first-GEMV input as
 * quantized B fragments (dbf_batched_frag_bytes(m, batch) bytes, made by dbf_batched_quantize from
 * an activation matrix or by the previous layer's finalize), and up to 4 "consumers" -- layers
 * that read this layer's output Y next -- whose fragments the finalize writes from Y exactly as
 * stored (times each consumer's input scale b): bitwise what dbf_batched_quantize would make from
 * Y, one kernel and one read of Y fewer per layer.  Consumer fragment buffers hold n columns. */
typedef struct {
  const void* b; /* the consumer layer's per-column input scale (scale_dtype), or NULL */
  void* frag;    /* its fragment buffer: dbf_batched_frag_bytes(n, batch) bytes */
} dbf_batched_consumer;
size_t dbf_batched_frag_bytes(int64_t cols, int64_t batch);
int dbf_batched_quantize(const void* X, int x_dtype, int64_t ldx, int64_t batch, int64_t cols,
                         const void* iscale, int scale_dtype, void* frag, void* stream);
size_t dbf_forward_batched_frag_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch);
/* Diagnostics (builds with -DDBF_BATCHED_TRACE, tools/batched_trace.py; DBF_ERR_UNSUPPORTED
 * otherwise): reset the per-launch trace slots (restart_slots != 0 also restarts their numbering),
 * and copy n slots of {kind (1 quantize, 2 GEMV, 3 finalize), first CTA start, last return from
 * the grid dependency wait, last warp end, last mid-kernel mark (quantize: inputs loaded;
 * finalize: y stored)} (%globaltimer ns). */
int dbf_batched_debug_reset(int restart_slots);
int dbf_batched_debug_trace(unsigned long long* host, int n);
int dbf_forward_batched_frag(const void* A_tiled, const void* B_tiled, const void* a,
                             const void* mid, int scale_dtype, int64_t n, int64_t k, int64_t m,
                             const void* frag_in, int64_t batch, void* Y, int y_dtype, int64_t ldy,
                             const dbf_batched_consumer* consumers, int nconsumers, void* workspace,
                             size_t workspace_bytes, unsigned* status, void* stream);

/* ---- prefill / batched path: tcgen05 + TMEM sign GEMMs (>= 64 tokens) ------------------ */
/*
 * The same forward as dbf_forward (kernel.py:48-62) for token batches, as two tensor-core GEMMs
 * with fp16 activations and fp32 accumulation in tensor memory:
 *   t = mid * (X . (B * b)^T)   (fp16 workspace, T x dbf_prefill_ld(k))
 *   Y = a   * (t . A^T)
 * Sign matrices are read in the PAIRED layout (dbf_pair_signs) and expanded to +-1 (times b for B)
 * on chip, straight into tensor memory.
 * Activations and scales are fp16; X must have ldx % 8 == 0 and a 16-byte aligned base
 * (DBF_ERR_UNSUPPORTED otherwise).  Not bitwise reproducible against dbf_forward: products
 * are exact, sums are fp32 and t is rounded to fp16 (DESIGN.md §5 tolerance).
 */
/* canonical words -> PAIRED prefill words (same pitch): per 32-column group, bit q (q < 16) holds
 * column 2q and bit 16+q column 2q+1, so one shift puts the signs of an fp16 pair at bits 15/31. */
int dbf_pair_signs(const uint32_t* words, int64_t rows, int64_t word_pitch, uint32_t* paired,
                   void* stream);
/* row pitch (elements) of the fp16 intermediate t in the prefill workspace */
int64_t dbf_prefill_ld(int64_t cols);
size_t dbf_prefill_workspace_bytes(int64_t k, int64_t tokens);
/* Workspace that also holds the split-K fp32 partials used for tokens <= 256 (the two GEMMs then
 * run over ~148 CTAs instead of rows/128; partials are summed in split order, deterministic).  A
 * workspace of only dbf_prefill_workspace_bytes runs the same GEMMs without splitting K. */
size_t dbf_prefill_workspace_bytes_nkm(int64_t n, int64_t k, int64_t m, int64_t tokens);

/* Diagnostics: with DBF_PREFILL_TRACE set in the environment, the last sign GEMM launch records
 * per-K-block clock64 stamps of CTA (0,0); copies n int64 of them to host memory. */
int dbf_prefill_debug_trace(long long* host, int n);

/* One sign GEMM: out[i, r] = rscale[r] * sum_c S[r, c] * kscale[c] * act[i, c]   (fp16 in/out)
 * act: tokens x K (stride ld_act), S: rows x K paired words, out: tokens x rows (stride ldo);
 * kscale / rscale may be NULL (= 1).  Replaces one staged sign_matvec of kernel.py:58-61. */
int dbf_sign_gemm(const void* act, int64_t tokens, int64_t K, int64_t ld_act, const uint32_t* paired,
                  int64_t word_pitch, int64_t rows, const void* kscale, const void* rscale, void* out,
                  int64_t ldo, void* stream);

/* kernel.forward (kernel.py:48-62) for a token batch: X tokens x m fp16 -> Y tokens x n fp16. */
int dbf_forward_prefill(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired,
                        int64_t B_pitch, const void* a, const void* mid, const void* b, int64_t n,
                        int64_t k, int64_t m, const void* X, int64_t tokens, int64_t ldx, void* Y,
                        int64_t ldy, void* workspace, size_t workspace_bytes, void* stream);

/* The same forward with an explicit kernel path.  DBF_PREFILL_TWO_LAUNCHES: one per-tile sign GEMM
 * launch per GEMM (T <= 256: split K).  DBF_PREFILL_ONE_LAUNCH (T > 256): both GEMMs in ONE persistent
 * launch, one CTA per SM claiming 128 x 256 tiles from a global counter, GEMM2 tiles of a token
 * block waiting on counters of its GEMM1 tiles; needs the workspace of dbf_prefill_workspace_bytes_nkm
 * (tile counters after t) and a TMA-compatible Y (ldy % 8 == 0, 16-byte aligned), else
 * DBF_ERR_UNSUPPORTED.  Both paths give bitwise identical outputs (same K order and rounding).
 * DBF_PREFILL_AUTO (what dbf_forward_prefill uses) = dbf_prefill_layer_path(n, k, m, tokens). */
enum { DBF_PREFILL_AUTO = 0, DBF_PREFILL_TWO_LAUNCHES = 1, DBF_PREFILL_ONE_LAUNCH = 2 };
int dbf_forward_prefill_ex(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired,
                           int64_t B_pitch, const void* a, const void* mid, const void* b, int64_t n,
                           int64_t k, int64_t m, const void* X, int64_t tokens, int64_t ldx, void* Y,
                           int64_t ldy, void* workspace, size_t workspace_bytes, int path, void* stream);
/* The path DBF_PREFILL_AUTO takes: one launch where GEMM1's tiles (k/128 x T/256) exceed the SM count
 * (a partly idle second wave), two launches otherwise (measured). */
int dbf_prefill_layer_path(int64_t n, int64_t k, int64_t m, int64_t tokens);


#ifdef __cplusplus
}
#endif
#endif /* DBF_B200_H */
