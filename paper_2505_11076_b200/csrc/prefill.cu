// DBF prefill / batched path (>= 64 tokens): the two sign GEMMs of one DBF forward on the
// 5th-generation tensor cores (tcgen05 + TMEM), replacing kernel.forward (kernel.py:48-62) for
// token batches where the layer is a real dense contraction:
//
//   GEMM1  t[T, k] = mid (.) ( X[T, m] . (B (.) b)^T )      B: k x m signs, b folded into B
//   GEMM2  Y[T, n] = a   (.) ( t[T, k] . A^T )              A: n x k signs
//
// One kernel, `sign_gemm_kernel`, runs either GEMM: out[T, rows] = rscale (.) (act . (S (.) kscale)^T)
// with S a rows x K sign matrix in the canonical word layout (include/dbf_b200.h).
//
// Per CTA: a 128 (sign rows) x 256 (tokens) output tile, accumulated in TMEM (256 fp32 columns).
//   warp 0       TMA producer: 256 x 64 fp16 activation tiles (128-byte swizzle) into a smem ring.
//   warp 1       TMEM allocator + MMA issuer (one thread): tcgen05.mma.kind::f16, M=128 N=256 K=16,
//                A operand from TMEM, B operand (activations) from shared memory.
//   warps 4..7   sign expanders, then epilogue.  Thread r owns sign row r of the tile (= TMEM
//                lane r): it reads the row's 64 packed bits per K block and writes 64 fp16 values
//                +-kscale[j] -- the fp16 sign bit XORed in from the packed bit -- straight into
//                TMEM with tcgen05.st (32x32b.x32).  No shared-memory traffic for the weights: the
//                +-1 expansion never leaves the tensor-memory side of the SM.
//   epilogue     tcgen05.ld of the accumulator (lane = sign row, column = token), scale by
//                rscale[row], fp16 store.
// The ring stage s couples a smem activation tile and a TMEM A slot; both are released by the
// tcgen05.commit of the MMAs that read them.
#include <cstring>
#include <mutex>
#include "common.cuh"
#include "sm100.cuh"

namespace dbf {
namespace prefill {

using namespace sm100;

constexpr int BM = 128;          // sign rows per tile (MMA M, TMEM lanes)
constexpr int BN = 256;          // tokens per tile (MMA N, accumulator columns)
constexpr int BK = 64;           // K per stage (one 128-byte swizzle atom of fp16)
constexpr int UK = 16;           // K per tcgen05.mma (kind::f16)
constexpr int STAGES = 4;
constexpr int kActStageBytes = BN * BK * 2;   // 32 KB
constexpr int kAColsPerStage = BK / 2;        // 32 TMEM columns (2 fp16 per 32-bit column)
constexpr int kAccCol = 0;
constexpr int kACol0 = BN;                    // A slots after the accumulator
constexpr int kTmemCols = 512;
constexpr int kThreads = 256;
constexpr int kExpWarp0 = 4;
static_assert(kACol0 + STAGES * kAColsPerStage <= kTmemCols, "TMEM budget");

struct Params {
  const uint32_t* words;   // rows x pitch canonical words
  int64_t pitch;           // words per row
  const __half* kscale;    // K values or nullptr (= 1)
  const __half* rscale;    // rows values or nullptr (= 1)
  __half* out;             // out[tok * ldo + row]
  int64_t ldo;
  int rows, K, T;
  int num_kb;
};

struct __align__(8) Barriers {
  uint64_t full_act[STAGES];
  uint64_t full_a[STAGES];
  uint64_t empty[STAGES];
  uint64_t acc_full;
  uint32_t tmem_base;
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + (size_t)STAGES * kActStageBytes + sizeof(Barriers);

// 64 packed signs (bit i = column i, 1 <=> +1) -> 32 words of fp16 pairs +-ks, in K order.
// Pair (2q, 2q+1) of the NEGATED bits moves to the fp16 sign positions 15 / 31 with one multiply:
// p * (2^(15-2q) + 2^(30-2q)) puts bit 2q at 15 and bit 2q+1 at 31 (no carries), then
// LOP3 ((prod & 0x80008000) ^ ks) applies it.
template <bool KSCALE>
__device__ __forceinline__ void expand_signs(uint64_t bits, const uint32_t* ks, uint32_t (&v)[32]) {
  const uint32_t nw[2] = {~(uint32_t)bits, ~(uint32_t)(bits >> 32)};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int half16 = 0; half16 < 2; ++half16) {
      const uint32_t w = half16 ? (nw[h] >> 16) : nw[h];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t p = w & (3u << (2 * q));
        const uint32_t mul = (1u << (15 - 2 * q)) + (1u << (30 - 2 * q));
        const int idx = h * 16 + half16 * 8 + q;
        const uint32_t base = KSCALE ? ks[idx] : 0x3C003C00u;
        v[idx] = ((p * mul) & 0x80008000u) ^ base;
      }
    }
  }
}

template <bool KSCALE>
__global__ void __launch_bounds__(kThreads, 1)
    sign_gemm_kernel(const __grid_constant__ CUtensorMap act_map, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* act = smem;
  Barriers& bar = *reinterpret_cast<Barriers*>(smem + (size_t)STAGES * kActStageBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * BM;
  const int tok0 = blockIdx.y * BN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bar.full_act[s], 1);
      mbar_init(&bar.full_a[s], 4);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&act_map);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // activations are re-read by every row tile
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&bar.empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar.full_act[s], kActStageBytes);
        tma_load_2d(act + (size_t)s * kActStageBytes, &act_map, kb * BK, tok0, &bar.full_act[s], pol);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(BM, BN);
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&bar.full_act[s], ph);
        mbar_wait(&bar.full_a[s], ph);
        tc_fence_after();
        const uint32_t a_base = tmem + kACol0 + s * kAColsPerStage;
        const uint32_t b_base = smem_u32(act + (size_t)s * kActStageBytes);
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          mma_f16_ts(tmem + kAccCol, a_base + kk * (UK / 2), sdesc_k_sw128(b_base + kk * UK * 2), idesc,
                     (kb | kk) != 0);
        }
        mma_commit(&bar.empty[s]);
      }
      mma_commit(&bar.acc_full);
    }
  } else if (warp >= kExpWarp0) {
    // ---------------- sign expanders + epilogue ----------------
    const int sub = warp & 3;                 // TMEM sub-partition this warp may access
    const int r = sub * 32 + lane;            // tile row = TMEM lane
    const int grow = row0 + r;
    const bool live = grow < p.rows;
    const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
    const uint32_t* wrow = p.words + (int64_t)(live ? grow : 0) * p.pitch;
    uint64_t next = live ? *(const uint64_t*)(wrow) : 0ull;
    for (int kb = 0; kb < p.num_kb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      const uint64_t bits = next;
      if (kb + 1 < p.num_kb && live) next = *(const uint64_t*)(wrow + 2 * (kb + 1));
      uint32_t ks[KSCALE ? 32 : 1];
      if constexpr (KSCALE) {
        const int c0 = kb * BK;
        if (c0 + BK <= p.K) {
          const uint4* src = reinterpret_cast<const uint4*>(p.kscale + c0);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint4 u = __ldg(src + i);
            ks[4 * i] = u.x, ks[4 * i + 1] = u.y, ks[4 * i + 2] = u.z, ks[4 * i + 3] = u.w;
          }
        } else {
          const unsigned short* src = reinterpret_cast<const unsigned short*>(p.kscale);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int c = c0 + 2 * i;
            const uint32_t lo16 = c < p.K ? src[c] : 0u, hi16 = c + 1 < p.K ? src[c + 1] : 0u;
            ks[i] = lo16 | (hi16 << 16);
          }
        }
      }
      uint32_t v[32];
      expand_signs<KSCALE>(bits, ks, v);
      mbar_wait(&bar.empty[s], ph ^ 1);
      tc_fence_after();
      tmem_st32(tmem + lane_addr + kACol0 + s * kAColsPerStage, v);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.full_a[s]);
    }
    // epilogue
    mbar_wait(&bar.acc_full, 0);
    tc_fence_after();
    const float rs = (live && p.rscale) ? __half2float(p.rscale[grow]) : 1.f;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t acc[32];
      tmem_ld32(tmem + lane_addr + kAccCol + c * 32, acc);
      tmem_wait_ld();
      if (live) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int tok = tok0 + c * 32 + j;
          if (tok < p.T) p.out[(int64_t)tok * p.ldo + grow] = __float2half_rn(__uint_as_float(acc[j]) * rs);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---- host side --------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// act: T x K fp16, row stride ld elements (ld*2 % 16 == 0, 16-byte aligned base)
static int make_act_map(CUtensorMap* map, const void* act, int64_t T, int64_t K, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return DBF_ERR_CUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {BK, BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(act), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? DBF_OK : DBF_ERR_CUDA;
}

static int launch_sign_gemm(const void* act, int64_t T, int64_t K, int64_t ld_act, const uint32_t* words,
                            int64_t pitch, int64_t rows, const __half* kscale, const __half* rscale, __half* out,
                            int64_t ldo, cudaStream_t stream) {
  if (T < 1 || K < 1 || rows < 1) return DBF_ERR_INVALID_ARGUMENT;
  if ((ld_act * 2) % 16 != 0 || ((uintptr_t)act & 15) != 0 || ld_act < K) return DBF_ERR_UNSUPPORTED;
  if (pitch * 32 < ceil_div(K, BK) * BK) return DBF_ERR_SHAPE;  // a K block would read past the row
  if (T > INT32_MAX || rows > INT32_MAX || K > INT32_MAX) return DBF_ERR_UNSUPPORTED;
  CUtensorMap map;
  int st = make_act_map(&map, act, T, K, ld_act);
  if (st != DBF_OK) return st;
  Params p;
  p.words = words;
  p.pitch = pitch;
  p.kscale = kscale;
  p.rscale = rscale;
  p.out = out;
  p.ldo = ldo;
  p.rows = (int)rows;
  p.K = (int)K;
  p.T = (int)T;
  p.num_kb = (int)ceil_div(K, BK);
  dim3 grid((unsigned)ceil_div(rows, BM), (unsigned)ceil_div(T, BN));
  if (kscale) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sign_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      attr = true;
    }
    sign_gemm_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(map, p);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sign_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      attr = true;
    }
    sign_gemm_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(map, p);
  }
  return check_launch();
}

}  // namespace prefill
}  // namespace dbf

using namespace dbf;

extern "C" {

int64_t dbf_prefill_ld(int64_t cols) { return ceil_div(cols, 64) * 64; }

size_t dbf_prefill_workspace_bytes(int64_t k, int64_t tokens) {
  return (size_t)(tokens > 0 ? tokens : 0) * (size_t)dbf_prefill_ld(k) * 2;
}

int dbf_sign_gemm(const void* act, int64_t tokens, int64_t K, int64_t ld_act, const uint32_t* words,
                  int64_t word_pitch, int64_t rows, const void* kscale, const void* rscale, void* out, int64_t ldo,
                  void* stream) {
  if (!act || !words || !out) return DBF_ERR_INVALID_ARGUMENT;
  if (ldo < rows) return DBF_ERR_SHAPE;
  return prefill::launch_sign_gemm(act, tokens, K, ld_act, words, word_pitch, rows, (const __half*)kscale,
                                   (const __half*)rscale, (__half*)out, ldo, (cudaStream_t)stream);
}

int dbf_forward_prefill(const uint32_t* A_words, int64_t A_pitch, const uint32_t* B_words, int64_t B_pitch,
                        const void* a, const void* mid, const void* b, int64_t n, int64_t k, int64_t m,
                        const void* X, int64_t tokens, int64_t ldx, void* Y, int64_t ldy, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!A_words || !B_words || !a || !mid || !b || !X || !Y) return DBF_ERR_INVALID_ARGUMENT;
  if (n < 1 || k < 1 || m < 1 || tokens < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (ldy < n || ldx < m) return DBF_ERR_SHAPE;
  if (A_pitch < canonical_pitch(k) || B_pitch < canonical_pitch(m)) return DBF_ERR_SHAPE;
  if (!workspace || workspace_bytes < dbf_prefill_workspace_bytes(k, tokens)) return DBF_ERR_WORKSPACE;
  const int64_t ldt = dbf_prefill_ld(k);
  __half* t = (__half*)workspace;
  cudaStream_t s = (cudaStream_t)stream;
  int st = prefill::launch_sign_gemm(X, tokens, m, ldx, B_words, B_pitch, k, (const __half*)b,
                                     (const __half*)mid, t, ldt, s);
  if (st != DBF_OK) return st;
  return prefill::launch_sign_gemm(t, tokens, k, ldt, A_words, A_pitch, n, nullptr, (const __half*)a,
                                   (__half*)Y, ldy, s);
}

}  // extern "C"
