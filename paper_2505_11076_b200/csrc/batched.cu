// Batched decode (2-16 tokens): kernel.forward (/root/reference/pkg/src/dbf/kernel.py:48-62) for a
// small token batch with ONE pass over each sign matrix for all tokens.
//
// The decode engine (engine.cu) carries at most 4 tokens per launch (4 tokens x 2 digit planes =
// the 8 columns of one IMMA.16832); larger batches used to re-stream the weights once per group of
// 4.  Here every extracted A fragment (one LOP3 per 4 weights, the engine's 2^t-bit trick) feeds
// NJ = ceil(batch / 4) IMMAs, one per token group, so the weights are read once per stage:
//
//   quantize   x (or the fp32 split partials of the previous stage, times its row scale) ->
//              per (token, 256-column chunk) 13-bit grid X = rint(u * 2^F * kQScale) (the
//              engine's numerics: |X| <= 4079), two balanced int8 digit planes of X * 2^(3-t)
//              in the IMMA B-fragment layout, F and T = sum X per (chunk, token)
//   gemv       one warp per 16-row block; for each 256-column chunk of its K range: the tiled
//              sign words (uint4 per lane), 8 k-blocks x NJ IMMAs (u8 x s8 -> s32), then
//              P = (s0 + 256 s1) / 4 - T (exact) and y += P / (2^F kQScale) in fp32;
//              K is split over gridDim.y CTAs (fp32 partials, summed in split order)
//   finalize   y = a (.) sum of the partials -> output dtype; non-finite / fp16-overflow status
//
// All layouts are the decode GEMV's (dbf_tile_signs); B fragments: bfrag[c][kb][j][lane] (uint2),
// lane = 8 * (token % 4) + 4 * plane + tig, bytes 0..3 = k 4*tig..+3, 4..7 = k 16+4*tig..+3.
#include <algorithm>
#include "common.cuh"
#include "sm100.cuh"

namespace dbf {
namespace batched {

constexpr int kWarps = 8;                 // quantize: (chunk, token) items per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kGemvWarps = 4;             // gemv: 16-row blocks per CTA (one per warp)
constexpr int kCtasPerSm = 8;             // gemv grid target (K splits fill it) ...
constexpr int kMaxSplits = 8;             // ... up to this many partials per output (the next
                                          // kernel sums them: more made that sum the long pole)
constexpr int kMaxTokens = 16;
constexpr float kQScale = 4079.f / 4096.f;  // 8 * |X| stays below the two-digit limit 32640
constexpr int kBadF = -128;                 // chunk holding inf / NaN: outputs it feeds are NaN
constexpr int kStatusNonFinite = 1, kStatusOverflow = 2;

__device__ __forceinline__ void imma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// weights: read once (no L1 allocation, evict-first in L2 so the activations stay resident)
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float load_f(const void* p, int dt, int64_t i) {
  switch (dt) {
    case DBF_F16: return __half2float(((const __half*)p)[i]);
    case DBF_F32: return ((const float*)p)[i];
    case DBF_F64: return (float)((const double*)p)[i];
    default: return __bfloat162float(((const __nv_bfloat16*)p)[i]);
  }
}
// Programmatic dependent launch: every kernel of a layer is launched with
// programmaticStreamSerialization, so it starts while its predecessor drains; it may only prefetch
// constant data (sign words, scales) before grid_wait(), which returns once the predecessor grid
// has completed and its memory is visible.  Reads AND writes of activations, fragments and partials
// come after it (the predecessor may still read what this kernel overwrites).
__device__ __forceinline__ void grid_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Input of one quantize launch: a row-major activation matrix (x, dtype, ldx) with an optional
// per-column scale, OR the fp32 split partials of the previous stage (part[s][t][cols], s < splits)
// with the previous stage's per-row scale (pscale) -- the two GEMVs of a layer chain through it.
struct QuantIn {
  const void* x;
  int x_dtype;
  int64_t ldx;
  const void* iscale;  // per column, scale_dtype, or null
  const float* part;    // part[s][t][ldx] (row stride ldx, a multiple of 4 floats)
  int splits;
  int64_t part_stride;  // floats between splits (= tpad * ldx)
  const void* pscale;   // per column of the partials (the previous GEMV's row scale), or null
  int scale_dtype;
  int cols, batch, tpad;
};

// One warp per (chunk, token): 64 groups of 4 columns, lane holds groups lane and lane + 32.
__global__ void __launch_bounds__(kThreads) quantize_kernel(QuantIn in, uint2* __restrict__ bfrag,
                                                            int* __restrict__ Fo, int* __restrict__ To, int nj) {
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nch = (in.cols + kChunkCols - 1) / kChunkCols;
  grid_wait();
  grid_launch_dependents();
  if (item >= nch * in.tpad) return;
  const int c = item / in.tpad, t = item % in.tpad;
  uint8_t* bf = reinterpret_cast<uint8_t*>(bfrag);
  if (t >= in.batch) {  // padding token: zero digits, F = T = 0 (its outputs are never stored)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = lane + 32 * h, kb = q >> 3, tig = q & 3, half = (q >> 2) & 1;
      uint8_t* base = bf + ((((size_t)c * 8 + kb) * nj + (t >> 2)) * 32 + 8 * (t & 3)) * 8 + 4 * half + tig * 8;
      *(uint32_t*)(base + 0) = 0u;
      *(uint32_t*)(base + 32) = 0u;
    }
    if (lane == 0) Fo[c * in.tpad + t] = 0, To[c * in.tpad + t] = 0;
    return;
  }
  float u[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j0 = c * kChunkCols + 4 * (lane + 32 * h);  // this lane's group of 4 columns
    float sc[4] = {1.f, 1.f, 1.f, 1.f};
    const void* scp = in.part ? in.pscale : in.iscale;
    if (j0 + 3 < in.cols) {
      if (in.part) {
        // the previous stage's split partials, summed in split order (deterministic); rows are
        // padded to a multiple of 4 floats (16-byte groups)
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int s = 0; s < in.splits; ++s) {
          const float4 b = __ldcg((const float4*)(in.part + (size_t)s * in.part_stride + (size_t)t * in.ldx + j0));
          a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
        }
        u[h][0] = a.x, u[h][1] = a.y, u[h][2] = a.z, u[h][3] = a.w;
      } else if (in.x_dtype == DBF_F16 && ((in.ldx | (int64_t)(uintptr_t)in.x / 2) & 3) == 0) {
        const uint2 r = __ldg((const uint2*)((const __half*)in.x + (int64_t)t * in.ldx + j0));
        const float2 lo = __half22float2(*(const __half2*)&r.x), hi = __half22float2(*(const __half2*)&r.y);
        u[h][0] = lo.x, u[h][1] = lo.y, u[h][2] = hi.x, u[h][3] = hi.y;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) u[h][e] = load_f(in.x, in.x_dtype, (int64_t)t * in.ldx + j0 + e);
      }
      if (scp) {
        if (in.scale_dtype == DBF_F16) {
          const uint2 r = __ldg((const uint2*)((const __half*)scp + j0));
          const float2 lo = __half22float2(*(const __half2*)&r.x), hi = __half22float2(*(const __half2*)&r.y);
          sc[0] = lo.x, sc[1] = lo.y, sc[2] = hi.x, sc[3] = hi.y;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) sc[e] = load_f(scp, in.scale_dtype, j0 + e);
        }
      }
    } else {  // the ragged end of the last chunk
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = j0 + e;
        float v = 0.f;
        if (j < in.cols) {
          if (in.part) {
            for (int s = 0; s < in.splits; ++s) v += __ldcg(in.part + (size_t)s * in.part_stride + (size_t)t * in.ldx + j);
          } else {
            v = load_f(in.x, in.x_dtype, (int64_t)t * in.ldx + j);
          }
          if (scp) sc[e] = load_f(scp, in.scale_dtype, j);
        }
        u[h][e] = v;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) u[h][e] *= sc[e];
  }
  float mx = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 4; ++e) mx = fmax_nan(mx, fabsf(u[h][e]));
  const uint32_t mxb = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
  int F = 0;
  float scale = 0.f;
  if (mxb >= 0x7F800000u) {
    F = kBadF;  // inf / NaN in the chunk: zero digits, NaN outputs
  } else {
    if (mxb != 0u) {
      const int ex = (int)(mxb >> 23) - 126;  // mx in [2^(ex-1), 2^ex)
      F = 12 - ex;
      F = F > 125 ? 125 : (F < -125 ? -125 : F);
    }
    scale = __int_as_float((F + 127) << 23) * kQScale;
  }
  int ts = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h, kb = q >> 3, tig = q & 3, half = (q >> 2) & 1;
    const int sh = 3 - (kb & 3);  // Y = X * 2^(3-t): the A bytes are 2^t * bit for k-block 4s + t
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int X = __float_as_int(fmaf(u[h][e], scale, 12582912.f)) - 0x4B400000;  // rint, |X| <= 4079
      ts += X;
      v[e] = (uint32_t)((X << sh) + 0x8080);  // bytes 0, 1 = balanced digits + 128
    }
    const uint32_t lo = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);
    uint8_t* base = bf + ((((size_t)c * 8 + kb) * nj + (t >> 2)) * 32 + 8 * (t & 3)) * 8 + 4 * half + tig * 8;
    *(uint32_t*)(base + 0) = lo ^ 0x80808080u;   // plane 0: MMA column 2 * (t % 4)
    *(uint32_t*)(base + 32) = hi ^ 0x80808080u;  // plane 1: MMA column 2 * (t % 4) + 1
  }
  ts = __reduce_add_sync(0xffffffffu, ts);
  if (lane == 0) Fo[c * in.tpad + t] = F, To[c * in.tpad + t] = ts;
}

struct GemvArgs {
  const uint4* tiled;  // rows x cols tiled signs
  int rows, nrb, nch, cps;  // cps: chunks per K split (gridDim.y splits)
  const uint2* bfrag;
  const int* F;
  const int* T;
  int tpad, batch;
  float* part;  // part[split][tpad][ldp]
  int ldp;      // partial row stride: rows rounded up to 4 floats
};

// One warp per 16-row block and K split; NJ token groups of 4 share every extracted A fragment.
// The chunk's B fragments (NJ x 2 KB, shared by the CTA's warps) stream through a 3-slot shared
// memory ring by bulk copy, two chunks ahead (loaded at use from L1 they were the whole stall
// profile: ~14 % L2 misses behind every IMMA); in registers the next k-block's fragments load
// while the current one's IMMAs run.  Sign words run two chunks ahead of the MMAs.
template <int NJ, int RB>
__global__ void __launch_bounds__(kGemvWarps * 32) gemv_kernel(GemvArgs g) {
  using namespace sm100;
  constexpr int kBBytes = 8 * NJ * 32 * 8;  // B fragments of one chunk
  constexpr int kSlots = 3;
  __shared__ __align__(128) uint8_t bsm[kSlots][kBBytes];
  __shared__ __align__(8) uint64_t full[kSlots], empty[kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb0 = (blockIdx.x * kGemvWarps + warp) * RB;  // this warp's RB row blocks
  const int c0 = blockIdx.y * g.cps, c1 = min(g.nch, c0 + g.cps), n = c1 - c0;
  const int gr = lane >> 2, tig = lane & 3;
  const uint64_t pol = evict_first_policy();
  const uint4* wb[RB];
  bool live[RB];
#pragma unroll
  for (int q = 0; q < RB; ++q) {
    live[q] = rb0 + q < g.nrb;  // a warp past the last row block still runs the ring (no stores)
    wb[q] = g.tiled + (int64_t)(live[q] ? rb0 + q : 0) * g.nch * 32 + lane;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], kGemvWarps);
    fence_mbar_init();
  }
  // the sign words are constant: their first chunks load while the previous kernel drains
  uint4 w[RB], wn[RB];
#pragma unroll
  for (int q = 0; q < RB; ++q) {
    w[q] = live[q] && n > 0 ? ld_stream(wb[q] + (int64_t)c0 * 32, pol) : make_uint4(0, 0, 0, 0);
    wn[q] = live[q] && n > 1 ? ld_stream(wb[q] + (int64_t)(c0 + 1) * 32, pol) : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  grid_wait();
  grid_launch_dependents();
  const uint8_t* bsrc = reinterpret_cast<const uint8_t*>(g.bfrag) + (size_t)c0 * kBBytes;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 && i < n; ++i) {
      mbar_arrive_expect_tx(&full[i], kBBytes);
      bulk_copy_g2s(bsm[i], bsrc + (size_t)i * kBBytes, kBBytes, &full[i]);
    }
  }
  float y[RB][NJ][2];
#pragma unroll
  for (int q = 0; q < RB; ++q)
#pragma unroll
    for (int j = 0; j < NJ; ++j) y[q][j][0] = y[q][j][1] = 0.f;
  for (int i = 0; i < n; ++i) {
    const int c = c0 + i, slot = i % kSlots;
    if (threadIdx.x == 0 && i + 2 < n) {  // chunk i + 2 into the slot chunk i - 1 held
      const int s2 = (i + 2) % kSlots;
      if (i + 2 >= kSlots) mbar_wait(&empty[s2], (((i + 2) / kSlots) - 1) & 1);
      mbar_arrive_expect_tx(&full[s2], kBBytes);
      bulk_copy_g2s(bsm[s2], bsrc + (size_t)(i + 2) * kBBytes, kBBytes, &full[s2]);
    }
    uint4 wnn[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q)
      wnn[q] = live[q] && i + 2 < n ? ld_stream(wb[q] + (int64_t)(c + 2) * 32, pol) : make_uint4(0, 0, 0, 0);
    int Fv[NJ], Tv[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) Fv[j] = __ldg(g.F + c * g.tpad + 4 * j + tig), Tv[j] = __ldg(g.T + c * g.tpad + 4 * j + tig);
    int acc[RB][NJ][4];
#pragma unroll
    for (int q = 0; q < RB; ++q)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[q][j][0] = acc[q][j][1] = acc[q][j][2] = acc[q][j][3] = 0;
    mbar_wait(&full[slot], (i / kSlots) & 1);
    const uint2* bf = reinterpret_cast<const uint2*>(bsm[slot]) + lane;
    uint2 bc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) bc[j] = bf[j * 32];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      uint2 bn[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bn[j] = r < 7 ? bf[((r + 1) * NJ + j) * 32] : make_uint2(0, 0);
      const uint32_t m = 0x01010101u << (r & 3);
      const int sh = r < 4 ? 0 : 4;
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const uint32_t a0 = (w[q].x >> sh) & m, a1 = (w[q].y >> sh) & m, a2 = (w[q].z >> sh) & m,
                       a3 = (w[q].w >> sh) & m;
#pragma unroll
        for (int j = 0; j < NJ; ++j) imma_u8s8(acc[q][j], a0, a1, a2, a3, bc[j].x, bc[j].y);
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) bc[j] = bn[j];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    // columns 2*tig, 2*tig+1 = token 4j + tig's two digit planes, rows gr and gr + 8
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int F = Fv[j], T = Tv[j];
      // P / (2^F kQScale) (exact P, |P| < 2^24); a chunk with inf / NaN (F = kBadF) makes the
      // outputs it feeds NaN
      const float inv = __int_as_float((127 - F) << 23) * (1.f / kQScale);
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const float p0 = (float)(((acc[q][j][0] + 256 * acc[q][j][1]) >> 2) - T);
        const float p1 = (float)(((acc[q][j][2] + 256 * acc[q][j][3]) >> 2) - T);
        y[q][j][0] = F == kBadF ? __int_as_float(0x7FC00000) : fmaf(p0, inv, y[q][j][0]);
        y[q][j][1] = F == kBadF ? __int_as_float(0x7FC00000) : fmaf(p1, inv, y[q][j][1]);
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) w[q] = wn[q], wn[q] = wnn[q];
  }
  float* out = g.part + (size_t)blockIdx.y * g.tpad * g.ldp;
#pragma unroll
  for (int q = 0; q < RB; ++q) {
    if (!live[q]) continue;
    const int row0 = (rb0 + q) * 16 + gr;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int t = 4 * j + tig;
      if (t < g.batch) {
        if (row0 < g.rows) out[(size_t)t * g.ldp + row0] = y[q][j][0];
        if (row0 + 8 < g.rows) out[(size_t)t * g.ldp + row0 + 8] = y[q][j][1];
      }
    }
  }
}

// y[t][r] = oscale[r] * sum_s part[s][t][r]  (split order), rounded to the output dtype; status
// bits: 1 = a non-finite value, 2 = a finite value beyond the fp16 range (fp16 output)
__global__ void finalize_kernel(const float* __restrict__ part, int splits, int64_t part_stride, int ldp, int rows,
                                int batch, const void* oscale, int scale_dtype, void* y, int y_dtype, int64_t ldy,
                                unsigned* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const float sc = (oscale && i < (int64_t)batch * rows) ? load_f(oscale, scale_dtype, i % rows) : 1.f;
  grid_wait();
  grid_launch_dependents();
  if (i >= (int64_t)batch * rows) return;
  const int t = (int)(i / rows), r = (int)(i % rows);
  float v = 0.f;
#pragma unroll 4
  for (int s = 0; s < splits; ++s) v += __ldcg(part + (size_t)s * part_stride + (size_t)t * ldp + r);
  v *= sc;
  const int64_t o = (int64_t)t * ldy + r;
  unsigned bad = isfinite(v) ? 0u : (unsigned)kStatusNonFinite;
  switch (y_dtype) {
    case DBF_F16: {
      const __half h = __float2half_rn(v);
      if (!bad && __hisinf(h)) bad = kStatusOverflow;
      ((__half*)y)[o] = h;
      break;
    }
    case DBF_F32: ((float*)y)[o] = v; break;
    case DBF_F64: ((double*)y)[o] = (double)v; break;
    default: ((__nv_bfloat16*)y)[o] = __float2bfloat16_rn(v); break;
  }
  if (bad && status) atomicOr(status, bad);
}

// ---- host side ---------------------------------------------------------------------------------
inline int tpad_of(int64_t batch) { return (int)ceil_div(batch, 4) * 4; }
inline int ldp_of(int64_t rows) { return (int)ceil_div(rows, 4) * 4; }
inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// row blocks per warp: two where there are enough rows (the chunk's B fragments, barriers and
// scale loads then serve twice the MMAs)
inline int rb_per_warp(int64_t nrb) { return nrb >= 128 ? 2 : 1; }
// K splits of one GEMV: enough CTAs for kCtasPerSm per SM, whole chunks per split
inline int split_count(int64_t nrb, int64_t nch, int* cps) {
  const int64_t gx = ceil_div(nrb, (int64_t)kGemvWarps * rb_per_warp(nrb));
  int64_t S = std::max<int64_t>(1, ceil_div((int64_t)kCtasPerSm * kNumSMs, gx));
  S = std::min<int64_t>(std::min<int64_t>(S, kMaxSplits), nch);
  const int64_t c = ceil_div(nch, S);
  *cps = (int)c;
  return (int)ceil_div(nch, c);
}

struct Layout {
  size_t bfrag, fo, to, part, total;
};
inline Layout layout_of(int64_t n, int64_t k, int64_t m, int64_t batch) {
  const int tpad = tpad_of(batch), nj = tpad / 4;
  const int64_t nchmax = std::max(chunks(m), chunks(k));
  int cps;
  const int S1 = split_count(row_blocks(k), chunks(m), &cps), S2 = split_count(row_blocks(n), chunks(k), &cps);
  Layout L;
  L.bfrag = 0;
  L.fo = align256(L.bfrag + (size_t)nchmax * 8 * nj * 32 * 8);
  L.to = align256(L.fo + (size_t)nchmax * tpad * 4);
  L.part = align256(L.to + (size_t)nchmax * tpad * 4);
  // stage-1 partials stay live while stage 2 quantizes from them: both sets side by side
  L.total = align256(L.part + ((size_t)S1 * tpad * ldp_of(k) + (size_t)S2 * tpad * ldp_of(n)) * 4 + 256);
  return L;
}

// every kernel of the chain: programmatic dependent launch (see grid_wait)
template <typename... KArgs, typename... Args>
static int launch_pdl(void (*kern)(KArgs...), dim3 grid, int threads, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  return check_launch();
}
template <int RB>
static int gemv_rb(const GemvArgs& a, int nj, int splits, cudaStream_t s) {
  const dim3 grid((unsigned)ceil_div(a.nrb, kGemvWarps * RB), (unsigned)splits);
  switch (nj) {
    case 1: return launch_pdl(gemv_kernel<1, RB>, grid, kGemvWarps * 32, s, a);
    case 2: return launch_pdl(gemv_kernel<2, RB>, grid, kGemvWarps * 32, s, a);
    case 3: return launch_pdl(gemv_kernel<3, RB>, grid, kGemvWarps * 32, s, a);
    default: return launch_pdl(gemv_kernel<4, RB>, grid, kGemvWarps * 32, s, a);
  }
}
static int gemv(const GemvArgs& a, int nj, int splits, cudaStream_t s) {
  return rb_per_warp(a.nrb) == 2 ? gemv_rb<2>(a, nj, splits, s) : gemv_rb<1>(a, nj, splits, s);
}

}  // namespace batched
}  // namespace dbf

using namespace dbf;

extern "C" {

size_t dbf_forward_batched_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch) {
  if (n < 1 || k < 1 || m < 1 || batch < 1 || batch > batched::kMaxTokens) return 0;
  return batched::layout_of(n, k, m, batch).total;
}

int dbf_forward_batched(const void* A_tiled, const void* B_tiled, const void* a, const void* mid, const void* b,
                        int scale_dtype, int64_t n, int64_t k, int64_t m, const void* X, int x_dtype, int64_t batch,
                        int64_t ldx, void* Y, int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes,
                        unsigned* status, void* stream) {
  using namespace batched;
  if (!A_tiled || !B_tiled || !X || !Y) return DBF_ERR_INVALID_ARGUMENT;
  if (n < 1 || k < 1 || m < 1 || batch < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (batch > kMaxTokens) return DBF_ERR_UNSUPPORTED;
  if (n > INT32_MAX / 2 || k > INT32_MAX / 2 || m > INT32_MAX / 2) return DBF_ERR_UNSUPPORTED;
  if (ldx < m || ldy < n) return DBF_ERR_SHAPE;
  if (!valid_float_dtype(x_dtype) || !valid_float_dtype(y_dtype) || !valid_float_dtype(scale_dtype))
    return DBF_ERR_INVALID_ARGUMENT;
  const Layout L = layout_of(n, k, m, batch);
  if (!workspace || workspace_bytes < L.total) return DBF_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  uint2* bfrag = (uint2*)(ws + L.bfrag);
  int* Fo = (int*)(ws + L.fo);
  int* To = (int*)(ws + L.to);
  const int tpad = tpad_of(batch), nj = tpad / 4;
  int cps1, cps2;
  const int S1 = split_count(row_blocks(k), chunks(m), &cps1), S2 = split_count(row_blocks(n), chunks(k), &cps2);
  const int ldk = ldp_of(k), ldn = ldp_of(n);
  float* part1 = (float*)(ws + L.part);
  float* part2 = part1 + (size_t)S1 * tpad * ldk;

  // stage 1: t = mid * (B . (x * b))
  QuantIn q{};
  q.x = X, q.x_dtype = x_dtype, q.ldx = ldx, q.iscale = b, q.scale_dtype = scale_dtype;
  q.cols = (int)m, q.batch = (int)batch, q.tpad = tpad;
  int st = launch_pdl(quantize_kernel, dim3((unsigned)ceil_div(chunks(m) * tpad, kWarps)), kThreads, s, q, bfrag,
                      Fo, To, nj);
  if (st != DBF_OK) return st;
  GemvArgs g1{(const uint4*)B_tiled, (int)k, (int)row_blocks(k), (int)chunks(m), cps1, bfrag, Fo, To, tpad,
              (int)batch, part1, ldk};
  if ((st = gemv(g1, nj, S1, s)) != DBF_OK) return st;
  // stage 2: y = a * (A . t), t quantized straight from the stage-1 partials
  QuantIn q2{};
  q2.part = part1, q2.splits = S1, q2.ldx = ldk, q2.part_stride = (int64_t)tpad * ldk, q2.pscale = mid;
  q2.scale_dtype = scale_dtype, q2.cols = (int)k, q2.batch = (int)batch, q2.tpad = tpad;
  st = launch_pdl(quantize_kernel, dim3((unsigned)ceil_div(chunks(k) * tpad, kWarps)), kThreads, s, q2, bfrag, Fo,
                  To, nj);
  if (st != DBF_OK) return st;
  GemvArgs g2{(const uint4*)A_tiled, (int)n, (int)row_blocks(n), (int)chunks(k), cps2, bfrag, Fo, To, tpad,
              (int)batch, part2, ldn};
  if ((st = gemv(g2, nj, S2, s)) != DBF_OK) return st;
  const int64_t total = batch * n;
  return launch_pdl(finalize_kernel, dim3((unsigned)ceil_div(total, 256)), 256, s, (const float*)part2, S2,
                    (int64_t)tpad * ldn, ldn, (int)n, (int)batch, a, scale_dtype, Y, y_dtype, ldy, status);
}

}  // extern "C"
