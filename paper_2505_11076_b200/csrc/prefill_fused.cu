// DBF prefill forward as ONE persistent kernel: both sign GEMMs of a layer,
//
//   GEMM1  t[T, k] = mid (.) ( X[T, m] . (B (.) b)^T )        (tiles 0 .. N1-1)
//   GEMM2  Y[T, n] = a   (.) ( t[T, k] . A^T )                (tiles N1 .. N1+N2-1)
//
// scheduled dynamically over one CTA per SM (a global tile counter), so the wave tail of GEMM1,
// the launch gap and GEMM2's ramp overlap: a GEMM2 tile of token block tb only waits until the
// k/128 GEMM1 tiles of tb have published t (per-token-block counters, release/acquire), which
// happens early because GEMM1 tiles are ordered token-block-major.  Tile mechanics follow
// prefill.cu (128 sign rows x 256 tokens, fp32 accumulator in TMEM, A = signs expanded straight
// into TMEM by 8 warps, B = activations by TMA); in addition the epilogue has its own 4 warps and
// a 64 KB staging tile stored by TMA, so it overlaps the next tile's mainloop (the MMA waits only
// for the accumulator to be drained into registers).
//
// Warp roles (16 warps): 0 scheduler + TMA producer, 1 TMEM allocator + MMA issuer, 4..11 sign
// expanders, 12..15 epilogue.  Spin loops carry a watchdog (__trap) so a broken dependency can
// never hang the GPU.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include "common.cuh"
#include "sm100.cuh"

namespace dbf {
namespace prefill_fused {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, UK = 16;
constexpr int kMaxStages = 6;
constexpr int kActStageBytes = BN * BK * 2;   // 32 KB
constexpr int kStageBytes = BN / 2 * BM * 2;  // 32 KB epilogue staging (fp16 [128 tokens][128 rows]), 2 halves per tile
constexpr int kAColsPerStage = BK / 2;
constexpr int kACol0 = BN;
constexpr int kTmemCols = 512;
constexpr int kExpWarp0 = 4, kExpWarps = 8, kEpiWarp0 = 12, kEpiWarps = 4;
constexpr int kThreads = 16 * 32;
constexpr int kTileRing = 4;
constexpr long long kSpinLimit = 1ll << 24;

struct Params {
  const uint32_t* B_words; int64_t B_pitch;   // k x m paired words
  const uint32_t* A_words; int64_t A_pitch;   // n x k paired words
  const __half* a; const __half* mid; const __half* b;
  int n, k, m, T;
  int rt1, rt2, tbs;       // row tiles of GEMM1 (k/128), GEMM2 (n/128), token blocks (T/256)
  int nkb1, nkb2;          // K blocks of GEMM1 (m/64), GEMM2 (k/64)
  int stages;
  int* sched;              // global tile counter (zeroed per call)
  int* done1;              // [tbs] GEMM1 tiles finished per token block (zeroed per call)
};

struct __align__(8) Bar {
  uint64_t full_act[kMaxStages], full_a[kMaxStages], empty[kMaxStages];
  uint64_t acc_full, acc_empty;
  uint64_t tile_full[kTileRing], tile_empty[kTileRing];
  int tile_id[kTileRing];
  uint32_t tmem_base;
};

constexpr size_t kBarBytes = (sizeof(Bar) + 127) / 128 * 128;

__device__ __forceinline__ void spin_guard(long long& n) {
  if (++n > kSpinLimit) __trap();
}
__device__ __forceinline__ void mbar_wait_guarded(uint64_t* bar, uint32_t parity) {
  long long n = 0;
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    spin_guard(n);
  }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}

__device__ __forceinline__ void expand_word(uint32_t w, const uint32_t* ks, uint32_t (&v)[16]) {
  const uint32_t nw = ~w;
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = ((nw << (15 - q)) & 0x80008000u) ^ ks[q];
}

struct TileInfo {
  int gemm;   // 1 or 2; 0 = no more tiles
  int rt, tb;
};
__device__ __forceinline__ TileInfo decode_tile(const Params& p, int t) {
  TileInfo ti;
  const int n1 = p.rt1 * p.tbs;
  if (t < n1) {
    ti.gemm = 1, ti.tb = t / p.rt1, ti.rt = t % p.rt1;
  } else if (t < n1 + p.rt2 * p.tbs) {
    t -= n1;
    ti.gemm = 2, ti.tb = t / p.rt2, ti.rt = t % p.rt2;
  } else {
    ti.gemm = 0, ti.tb = 0, ti.rt = 0;
  }
  return ti;
}

__global__ void __launch_bounds__(kThreads, 1)
    fused_kernel(const __grid_constant__ CUtensorMap x_map, const __grid_constant__ CUtensorMap t_map,
                 const __grid_constant__ CUtensorMap t_store, const __grid_constant__ CUtensorMap y_store,
                 const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* act = smem;
  uint8_t* stage_out = smem + (size_t)p.stages * kActStageBytes;
  Bar& bar = *reinterpret_cast<Bar*>(stage_out + kStageBytes);
  uint32_t* ks_smem = reinterpret_cast<uint32_t*>(stage_out + kStageBytes + kBarBytes);  // 16-byte aligned

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&bar.full_act[s], 1);
      mbar_init(&bar.full_a[s], kExpWarps);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc_full, 1);
    mbar_init(&bar.acc_empty, kEpiWarps);
    for (int j = 0; j < kTileRing; ++j) {
      mbar_init(&bar.tile_full[j], 1);
      mbar_init(&bar.tile_empty[j], 1 + kExpWarps + kEpiWarps);  // MMA thread + expander + epilogue warps
    }
    fence_mbar_init();
    tma_prefetch_desc(&x_map);
    tma_prefetch_desc(&t_map);
    tma_prefetch_desc(&t_store);
    tma_prefetch_desc(&y_store);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&bar.tmem_base);
  {  // b as fp16 pairs (GEMM1's K scale), zero beyond m
    const unsigned short* src = reinterpret_cast<const unsigned short*>(p.b);
    for (int i = threadIdx.x; i < p.nkb1 * (BK / 2); i += kThreads) {
      const int c = 2 * i;
      const uint32_t lo = c < p.m ? src[c] : 0u, hi = c + 1 < p.m ? src[c + 1] : 0u;
      ks_smem[i] = lo | (hi << 16);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  if (warp == 0) {
    // ---------------- scheduler + TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      int g = 0;  // global K-block counter (ring position)
      for (int j = 0;; ++j) {
        const int slot = j % kTileRing;
        mbar_wait_guarded(&bar.tile_empty[slot], ((j / kTileRing) & 1) ^ 1);
        const int t = atomicAdd(p.sched, 1);
        bar.tile_id[slot] = t;
        mbar_arrive(&bar.tile_full[slot]);
        const TileInfo ti = decode_tile(p, t);
        if (ti.gemm == 0) break;
        const CUtensorMap* map = ti.gemm == 1 ? &x_map : &t_map;
        const int nkb = ti.gemm == 1 ? p.nkb1 : p.nkb2;
        if (ti.gemm == 2) {  // t of this token block must be complete (GEMM1 epilogues)
          long long n = 0;
          while (true) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.done1 + ti.tb) : "memory");
            if (v >= p.rt1) break;
            __nanosleep(64);
            spin_guard(n);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          const uint32_t ph = (g / S) & 1;
          mbar_wait_guarded(&bar.empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&bar.full_act[s], kActStageBytes);
          tma_load_2d(act + (size_t)s * kActStageBytes, map, kb * BK, ti.tb * BN, &bar.full_act[s], pol);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(BM, BN);
      int g = 0;
      for (int j = 0;; ++j) {
        const int slot = j % kTileRing;
        mbar_wait_guarded(&bar.tile_full[slot], (j / kTileRing) & 1);
        const int t = bar.tile_id[slot];
        mbar_arrive(&bar.tile_empty[slot]);
        const TileInfo ti = decode_tile(p, t);
        if (ti.gemm == 0) break;
        const int nkb = ti.gemm == 1 ? p.nkb1 : p.nkb2;
        mbar_wait_guarded(&bar.acc_empty, (j & 1) ^ 1);  // the epilogue drained the accumulator
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          const uint32_t ph = (g / S) & 1;
          mbar_wait_guarded(&bar.full_act[s], ph);
          mbar_wait_guarded(&bar.full_a[s], ph);
          tc_fence_after();
          const uint32_t a_base = tmem + kACol0 + s * kAColsPerStage;
          const uint32_t b_base = smem_u32(act + (size_t)s * kActStageBytes);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk)
            mma_f16_ts(tmem, a_base + kk * (UK / 2), sdesc_k_sw128(b_base + kk * UK * 2), idesc, (kb | kk) != 0);
          mma_commit(&bar.empty[s]);
        }
        mma_commit(&bar.acc_full);
      }
    }
  } else if (warp >= kExpWarp0 && warp < kExpWarp0 + kExpWarps) {
    // ---------------- sign expanders ----------------
    const int sub = warp & 3, half = (warp - kExpWarp0) >> 2;
    const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
    int g = 0;
    for (int j = 0;; ++j) {
      const int slot = j % kTileRing;
      if (lane == 0) mbar_wait_guarded(&bar.tile_full[slot], (j / kTileRing) & 1);
      __syncwarp();
      const int t = bar.tile_id[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.tile_empty[slot]);
      const TileInfo ti = decode_tile(p, t);
      if (ti.gemm == 0) break;
      const bool g1 = ti.gemm == 1;
      const int rows = g1 ? p.k : p.n, nkb = g1 ? p.nkb1 : p.nkb2;
      const int grow = ti.rt * BM + sub * 32 + lane;
      const bool live = grow < rows;
      const uint4* wrow = reinterpret_cast<const uint4*>((g1 ? p.B_words : p.A_words) +
                                                         (int64_t)(live ? grow : 0) * (g1 ? p.B_pitch : p.A_pitch));
      const int nquads = (nkb + 1) >> 1;
      uint4 cur = make_uint4(0, 0, 0, 0), nxt = live ? __ldg(wrow) : make_uint4(0, 0, 0, 0);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S;
        const uint32_t ph = (g / S) & 1;
        if ((kb & 1) == 0) {
          cur = nxt;
          if (live && (kb >> 1) + 1 < nquads) nxt = __ldg(wrow + (kb >> 1) + 1);
        }
        const uint32_t w = (kb & 1) ? (half ? cur.w : cur.z) : (half ? cur.y : cur.x);
        uint32_t ks[16];
        if (g1) {
          const uint4* src = reinterpret_cast<const uint4*>(ks_smem + kb * (BK / 2) + half * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 u = src[i];
            ks[4 * i] = u.x, ks[4 * i + 1] = u.y, ks[4 * i + 2] = u.z, ks[4 * i + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) ks[i] = 0x3C003C00u;
        }
        uint32_t v[16];
        expand_word(w, ks, v);
        if (lane == 0) mbar_wait_guarded(&bar.empty[s], ph ^ 1);
        __syncwarp();
        tc_fence_after();
        tmem_st16(tmem + lane_addr + kACol0 + s * kAColsPerStage + half * 16, v);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.full_a[s]);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue ----------------
    const int sub = warp & 3;
    const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
    const int r = sub * 32 + lane;  // tile row
    __half* st = reinterpret_cast<__half*>(stage_out);
    for (int j = 0;; ++j) {
      const int slot = j % kTileRing;
      if (lane == 0) mbar_wait_guarded(&bar.tile_full[slot], (j / kTileRing) & 1);
      __syncwarp();
      const int t = bar.tile_id[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.tile_empty[slot]);
      const TileInfo ti = decode_tile(p, t);
      if (ti.gemm == 0) break;
      const bool g1 = ti.gemm == 1;
      const int rows = g1 ? p.k : p.n;
      const int grow = ti.rt * BM + r;
      const float rs = grow < rows ? __half2float((g1 ? p.mid : p.a)[grow]) : 0.f;
      if (lane == 0) mbar_wait_guarded(&bar.acc_full, j & 1);
      __syncwarp();
      tc_fence_after();
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {  // tokens [128*hh, 128*hh + 128) through the staging tile
        // the previous store must have read the staging buffer
        if (threadIdx.x == kEpiWarp0 * 32) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"n"(kEpiWarps * 32) : "memory");
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          uint32_t acc[32];
          tmem_ld32(tmem + lane_addr + hh * (BN / 2) + c * 32, acc);
          tmem_wait_ld();
          if (hh == 1 && c == BN / 64 - 1) {  // accumulator drained: the next tile's MMAs may start
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.acc_empty);
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) st[(c * 32 + e) * BM + r] = __float2half_rn(__uint_as_float(acc[e]) * rs);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (threadIdx.x == kEpiWarp0 * 32) {
          tma_store_2d(g1 ? &t_store : &y_store, st, ti.rt * BM, ti.tb * BN + hh * (BN / 2));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (threadIdx.x == kEpiWarp0 * 32 && g1) {  // publish t of this tile before counting it done
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.done1 + ti.tb) : "memory");
      }
    }
    if (threadIdx.x == kEpiWarp0 * 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---- host ------------------------------------------------------------------------------------
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
// fp16 matrix rows x inner (stride ld elements) with a box of box_inner x box_rows
static bool make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t rows, int64_t ld, int box_inner,
                     int box_rows, bool swizzle) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace prefill_fused
}  // namespace dbf

using namespace dbf;

extern "C" {

size_t dbf_prefill_fused_workspace_bytes(int64_t k, int64_t tokens) {
  const int64_t ldt = ceil_div(k, 64) * 64;
  return (size_t)tokens * (size_t)ldt * 2 + 256 + (size_t)ceil_div(tokens, 256) * 4 + 256;
}

int dbf_forward_prefill_fused(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired, int64_t B_pitch,
                              const void* a, const void* mid, const void* b, int64_t n, int64_t k, int64_t m,
                              const void* X, int64_t tokens, int64_t ldx, void* Y, int64_t ldy, void* workspace,
                              size_t workspace_bytes, void* stream) {
  using namespace prefill_fused;
  if (!A_paired || !B_paired || !a || !mid || !b || !X || !Y || !workspace) return DBF_ERR_INVALID_ARGUMENT;
  if (n < 1 || k < 1 || m < 1 || tokens < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (ldy < n || ldx < m) return DBF_ERR_SHAPE;
  if (A_pitch < canonical_pitch(k) || B_pitch < canonical_pitch(m) || A_pitch % 4 || B_pitch % 4)
    return DBF_ERR_SHAPE;
  if (workspace_bytes < dbf_prefill_fused_workspace_bytes(k, tokens)) return DBF_ERR_WORKSPACE;
  if ((ldx * 2) % 16 || ((uintptr_t)X & 15) || (ldy * 2) % 16 || ((uintptr_t)Y & 15) || ((uintptr_t)workspace & 255))
    return DBF_ERR_UNSUPPORTED;
  if (tokens > INT32_MAX || n > INT32_MAX || k > INT32_MAX || m > INT32_MAX) return DBF_ERR_UNSUPPORTED;
  const int64_t ldt = ceil_div(k, 64) * 64;
  __half* t = (__half*)workspace;
  uint8_t* ctr = (uint8_t*)workspace + ((size_t)tokens * ldt * 2 + 255) / 256 * 256;
  Params p;
  p.B_words = B_paired, p.B_pitch = B_pitch, p.A_words = A_paired, p.A_pitch = A_pitch;
  p.a = (const __half*)a, p.mid = (const __half*)mid, p.b = (const __half*)b;
  p.n = (int)n, p.k = (int)k, p.m = (int)m, p.T = (int)tokens;
  p.rt1 = (int)ceil_div(k, BM), p.rt2 = (int)ceil_div(n, BM), p.tbs = (int)ceil_div(tokens, BN);
  p.nkb1 = (int)ceil_div(m, BK), p.nkb2 = (int)ceil_div(k, BK);
  p.sched = (int*)ctr;
  p.done1 = (int*)(ctr + 16);
  const size_t ks_bytes = (size_t)p.nkb1 * BK * 2;
  const size_t fixed = 1024 + kStageBytes + kBarBytes + ks_bytes;
  const size_t max_smem = 227 * 1024;
  if (fixed + 2 * kActStageBytes > max_smem) return DBF_ERR_UNSUPPORTED;
  p.stages = (int)std::min<size_t>(kMaxStages, (max_smem - fixed) / kActStageBytes);
  const size_t smem = fixed + (size_t)p.stages * kActStageBytes;
  CUtensorMap xm, tm, ts, ys;
  if (!make_map(&xm, X, m, tokens, ldx, BK, BN, true) || !make_map(&tm, t, k, tokens, ldt, BK, BN, true) ||
      !make_map(&ts, t, k, tokens, ldt, BM, BN / 2, false) || !make_map(&ys, Y, n, tokens, ldy, BM, BN / 2, false))
    return DBF_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(ctr, 0, 16 + (size_t)p.tbs * 4, s);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem);
    if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tiles = (p.rt1 + p.rt2) * p.tbs;
  fused_kernel<<<std::min(sms, tiles), kThreads, smem, s>>>(xm, tm, ts, ys, p);
  return check_launch();
}

}  // extern "C"
