// Batched decode (2-32 tokens): kernel.forward (/root/reference/pkg/src/dbf/kernel.py:48-62) for a
// small token batch with ONE pass over each sign matrix for all tokens.
//
// The decode engine (engine.cu) carries at most 4 tokens per launch (4 tokens x 2 digit planes =
// the 8 columns of one IMMA.16832); larger batches used to re-stream the weights once per group of
// 4.  Here every extracted A fragment (one LOP3 per 4 weights, the engine's 2^t-bit trick) feeds
// NJ = ceil(batch / 4) IMMAs, one per token group, so the weights are read once per stage.  Four
// kernels per layer, each launched with programmatic dependent launch (it loads its sign words and
// scales while the previous kernel drains, then griddepcontrol.wait):
//
//   quantize   x, or the fp32 split partials of the first GEMV times mid -> per (token, 256-column
//              chunk) 13-bit grid X = rint(u * 2^F * kQScale) (the engine's numerics: |X| <=
//              4079), two balanced int8 digit planes of X * 2^(3-t) in the IMMA B-fragment
//              layout, F and T = sum X per (chunk, token)
//   gemv       one warp per one or two 16-row blocks; per 256-column chunk of its K range: the
//              tiled sign words (uint4 per lane, two chunks ahead), the chunk's B fragments from a
//              shared-memory ring filled by bulk copy, 8 k-blocks x NJ IMMAs (u8 x s8 -> s32),
//              P = (s0 + 256 s1) / 4 - T (exact) and y += P / (2^F kQScale) in fp32; K split
//              over gridDim.y CTAs (fp32 partials, summed in split order)
//   finalize   y = a (.) sum of the partials -> output dtype (status bits: non-finite, fp16
//              overflow), and the first-GEMV fragments of the layers that read y next (a layer
//              chain needs the standalone quantize only for inputs from outside it)
//
// Sign words: the decode GEMV's tiled layout (dbf_tile_signs).  B fragments: bfrag[c][kb][j][lane]
// (uint2), j = token / 4, lane = 8 * (token % 4) + 4 * plane + tig, bytes 0..3 = k 4*tig..+3,
// 4..7 = k 16+4*tig..+3.
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
constexpr int kMaxTokens = 32;
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

// Diagnostics build only (-DDBF_BATCHED_TRACE, tools/batched_trace.py): per launch slot, the
// earliest CTA start, the latest return from grid_wait and the latest CTA end (%globaltimer ns)
#ifdef DBF_BATCHED_TRACE
__device__ unsigned long long g_btrace[8192][5];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BT_START(slot) const unsigned long long bt0_ = gtime();
#define BT_WAITED(slot)                                                        \
  if ((slot) >= 0 && threadIdx.x == 0) {                                       \
    atomicMin(&g_btrace[slot][1], bt0_);                                       \
    atomicMax(&g_btrace[slot][2], gtime());                                    \
  }
#define BT_END(slot)                                                           \
  if ((slot) >= 0 && (threadIdx.x & 31) == 0) atomicMax(&g_btrace[slot][3], gtime());
#define BT_MARK(slot)                                                          \
  if ((slot) >= 0 && (threadIdx.x & 31) == 0) atomicMax(&g_btrace[slot][4], gtime());
#else
#define BT_MARK(slot)
#define BT_START(slot)
#define BT_WAITED(slot)
#define BT_END(slot)
#endif
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
  int tslot;  // diagnostics: trace slot (DBF_BATCHED_TRACE builds), -1
};

// Fragment buffer of one GEMV input (cols columns, tpad token slots): B fragments, then F, then T
struct FragView {
  uint2* bfrag;
  int* F;
  int* T;
};
inline size_t frag_bfrag_bytes(int64_t cols, int tpad) { return (size_t)chunks(cols) * 8 * (tpad / 4) * 32 * 8; }
inline size_t frag_bytes(int64_t cols, int tpad) {
  return ((frag_bfrag_bytes(cols, tpad) + 2 * (size_t)chunks(cols) * tpad * 4) + 255) & ~(size_t)255;
}
__host__ __device__ inline FragView frag_view(void* base, int64_t cols, int tpad) {
  FragView v;
  v.bfrag = (uint2*)base;
  const size_t fb = (size_t)((cols + kChunkCols - 1) / kChunkCols) * 8 * (tpad / 4) * 32 * 8;
  v.F = (int*)((char*)base + fb);
  v.T = v.F + (size_t)((cols + kChunkCols - 1) / kChunkCols) * tpad;
  return v;
}

// Padding token t of chunk c: zero digits, F = T = 0 (its outputs are never stored)
__device__ __forceinline__ void zero_chunk(int c, int t, const FragView& fv, int tpad, int nj) {
  const int lane = threadIdx.x & 31;
  uint8_t* bf = reinterpret_cast<uint8_t*>(fv.bfrag);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h, kb = q >> 3, tig = q & 3, half = (q >> 2) & 1;
    uint8_t* base = bf + ((((size_t)c * 8 + kb) * nj + (t >> 2)) * 32 + 8 * (t & 3)) * 8 + 4 * half + tig * 8;
    *(uint32_t*)(base + 0) = 0u;
    *(uint32_t*)(base + 32) = 0u;
  }
  if (lane == 0) fv.F[c * tpad + t] = 0, fv.T[c * tpad + t] = 0;
}

// Chunk c of token t (this lane: columns 4 (lane + 32 h) + e of the chunk, u already scaled) ->
// the 13-bit grid, two balanced digit planes in the B-fragment layout, F and T = sum X.
__device__ __forceinline__ void emit_chunk(const float (&u)[2][4], int c, int t, const FragView& fv, int tpad,
                                           int nj) {
  const int lane = threadIdx.x & 31;
  uint8_t* bf = reinterpret_cast<uint8_t*>(fv.bfrag);
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
  if (lane == 0) fv.F[c * tpad + t] = F, fv.T[c * tpad + t] = ts;
}

// One warp per (chunk, token): 64 groups of 4 columns, lane holds groups lane and lane + 32.
// 4 consecutive scale values (fp16 pairs loaded as one 8-byte word where aligned)
__device__ __forceinline__ void load_scale4(const void* p, int dt, int j0, float (&sc)[4]) {
  if (dt == DBF_F16 && (j0 & 3) == 0) {
    const uint2 r = __ldg((const uint2*)((const __half*)p + j0));
    const float2 lo = __half22float2(*(const __half2*)&r.x), hi = __half22float2(*(const __half2*)&r.y);
    sc[0] = lo.x, sc[1] = lo.y, sc[2] = hi.x, sc[3] = hi.y;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) sc[e] = load_f(p, dt, j0 + e);
  }
}

// the scales of columns j0..j0+3 (1 past the end / without a scale)
__device__ __forceinline__ void scale4_at(const void* p, int dt, int j0, int cols, float (&sc)[4]) {
  sc[0] = sc[1] = sc[2] = sc[3] = 1.f;
  if (!p) return;
  if (j0 + 3 < cols) {
    load_scale4(p, dt, j0, sc);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j0 + e < cols) sc[e] = load_f(p, dt, j0 + e);
  }
}
// sum of the split partials of columns j0..j0+3 of token row t, in split order; every split's
// 16-byte load is issued before the first add (one L2 round trip, not one per split)
__device__ __forceinline__ void sum_splits4(const float* part, int splits, int64_t stride, int64_t row_off, int j0,
                                            int cols, float (&v)[4]) {
  v[0] = v[1] = v[2] = v[3] = 0.f;
  if (j0 + 3 < cols) {
    float4 p[kMaxSplits];
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s)
      p[s] = s < splits ? __ldcg((const float4*)(part + (size_t)s * stride + row_off + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s)
      if (s < splits) v[0] += p[s].x, v[1] += p[s].y, v[2] += p[s].z, v[3] += p[s].w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j0 + e < cols)
        for (int s = 0; s < splits; ++s) v[e] += __ldcg(part + (size_t)s * stride + row_off + j0 + e);
  }
}
// 16-byte L2 load (ld.global.cg) the compiler keeps in program order: the two groups' loads of
// every split below go out back to back (left to the compiler, they went out two or three at a
// time, one L2 round trip each: 2.3 us to load a chunk's partials, tools/batched_trace.py)
__device__ __forceinline__ float4 ldcg4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// this lane's two groups (columns j0 .. j0+3 for j0 = ja, jb) of token row t summed over the
// splits in split order; all loads issued before the first add
__device__ __forceinline__ void sum_splits4x2(const float* part, int splits, int64_t stride, int64_t row_off, int ja,
                                              int jb, int cols, float (&va)[4], float (&vb)[4]) {
  if (ja + 3 < cols && jb + 3 < cols) {
    float4 pa[kMaxSplits], pb[kMaxSplits];
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s) {
      if (s < splits) {
        pa[s] = ldcg4(part + (size_t)s * stride + row_off + ja);
        pb[s] = ldcg4(part + (size_t)s * stride + row_off + jb);
      }
    }
    va[0] = va[1] = va[2] = va[3] = vb[0] = vb[1] = vb[2] = vb[3] = 0.f;
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s)
      if (s < splits) {
        va[0] += pa[s].x, va[1] += pa[s].y, va[2] += pa[s].z, va[3] += pa[s].w;
        vb[0] += pb[s].x, vb[1] += pb[s].y, vb[2] += pb[s].z, vb[3] += pb[s].w;
      }
    return;
  }
  sum_splits4(part, splits, stride, row_off, ja, cols, va);
  sum_splits4(part, splits, stride, row_off, jb, cols, vb);
}

// One warp per (chunk, token): 64 groups of 4 columns, lane holds groups lane and lane + 32.
__global__ void __launch_bounds__(kThreads) quantize_kernel(QuantIn in, FragView fv, int nj) {
  BT_START(in.tslot)
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nch = (in.cols + kChunkCols - 1) / kChunkCols;
  const int c = item / in.tpad, t = item % in.tpad;
  const bool live = item < nch * in.tpad && t < in.batch;
  // the column scales are constant: loaded while the previous kernel drains
  float sc[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
    scale4_at(live ? (in.part ? in.pscale : in.iscale) : nullptr, in.scale_dtype, c * kChunkCols + 4 * (lane + 32 * h),
              in.cols, sc[h]);
  grid_wait();
  BT_WAITED(in.tslot)
  grid_launch_dependents();
  if (item >= nch * in.tpad) return;
  if (t >= in.batch) {
    zero_chunk(c, t, fv, in.tpad, nj);
    return;
  }
  float u[2][4];
  if (in.part)  // the previous stage's split partials (rows padded to 4 floats), in split order
    sum_splits4x2(in.part, in.splits, in.part_stride, (int64_t)t * in.ldx, c * kChunkCols + 4 * lane,
                  c * kChunkCols + 4 * (lane + 32), in.cols, u[0], u[1]);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j0 = c * kChunkCols + 4 * (lane + 32 * h);  // this lane's group of 4 columns
    if (in.part) {
    } else if (j0 + 3 < in.cols && in.x_dtype == DBF_F16 && ((in.ldx | (int64_t)(uintptr_t)in.x / 2) & 3) == 0) {
      const uint2 r = __ldg((const uint2*)((const __half*)in.x + (int64_t)t * in.ldx + j0));
      const float2 lo = __half22float2(*(const __half2*)&r.x), hi = __half22float2(*(const __half2*)&r.y);
      u[h][0] = lo.x, u[h][1] = lo.y, u[h][2] = hi.x, u[h][3] = hi.y;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) u[h][e] = j0 + e < in.cols ? load_f(in.x, in.x_dtype, (int64_t)t * in.ldx + j0 + e) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) u[h][e] *= sc[h][e];
  }
  BT_MARK(in.tslot)
  emit_chunk(u, c, t, fv, in.tpad, nj);
  BT_END(in.tslot)
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
  int tslot;    // diagnostics: trace slot (DBF_BATCHED_TRACE builds), -1
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
  // ring depth: 3 slots (2 chunks ahead); 2 at NJ > 4 (16 KB slots, static shared memory)
  constexpr int kSlots = NJ > 4 ? 2 : 3, kAhead = kSlots - 1;
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
  BT_START(g.tslot)
  grid_wait();
  BT_WAITED(g.tslot)
  grid_launch_dependents();
  const uint8_t* bsrc = reinterpret_cast<const uint8_t*>(g.bfrag) + (size_t)c0 * kBBytes;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kAhead && i < n; ++i) {
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
    if (threadIdx.x == 0 && i + kAhead < n) {  // chunk i + kAhead into the slot chunk i - 1 held
      const int ia = i + kAhead, s2 = ia % kSlots;
      if (ia >= kSlots) mbar_wait(&empty[s2], ((ia / kSlots) - 1) & 1);
      mbar_arrive_expect_tx(&full[s2], kBBytes);
      bulk_copy_g2s(bsm[s2], bsrc + (size_t)ia * kBBytes, kBBytes, &full[s2]);
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
  BT_END(g.tslot)
}

// Layers that read this layer's output next (DecodePlan chains): each gets its first-GEMV B
// fragments straight from the finalize, from the output exactly as rounded to the output dtype and
// times its own input scale b -- bitwise what quantize_kernel would make from the stored output.
constexpr int kMaxConsumers = 4;
struct Consumer {
  const void* b;  // the consumer's per-column input scale (scale_dtype) or null
  FragView fv;
};
struct FinArgs {
  const float* part;  // part[s][tpad][ldp]
  int splits;
  int64_t part_stride;
  int ldp, rows, batch, tpad, nj;
  const void* oscale;
  int scale_dtype;
  void* y;
  int y_dtype;
  int64_t ldy;
  unsigned* status;
  int ncons;
  Consumer cons[kMaxConsumers];
  int tslot;  // diagnostics: trace slot (DBF_BATCHED_TRACE builds), -1
};

// One warp per (256-row chunk, token, consumer): y = oscale (.) sum of the splits (split order),
// rounded to the output dtype; the consumer-0 warp stores it and reports status bits 1 (a
// non-finite value) and 2 (a finite value beyond the fp16 range, fp16 output); every warp then
// writes its consumer's B fragments of the chunk (one warp per consumer: the chunk's rounding is
// recomputed, not shared, so the consumers run side by side).
__global__ void __launch_bounds__(kThreads) finalize_kernel(FinArgs f) {
  BT_START(f.tslot)
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nch = (f.rows + kChunkCols - 1) / kChunkCols, ncw = f.ncons > 0 ? f.ncons : 1;
  const int k = item % ncw, ct = item / ncw, c = ct / f.tpad, t = ct % f.tpad;
  const bool live = item < nch * f.tpad * ncw && t < f.batch;
  // the output scale and this warp's consumer's input scale are constant: loaded while the
  // previous kernel drains
  float osc[2][4], csc[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j0 = c * kChunkCols + 4 * (lane + 32 * h);
    scale4_at(live ? f.oscale : nullptr, f.scale_dtype, j0, f.rows, osc[h]);
    scale4_at(live && f.ncons > 0 ? f.cons[k].b : nullptr, f.scale_dtype, j0, f.rows, csc[h]);
  }
  grid_wait();
  BT_WAITED(f.tslot)
  grid_launch_dependents();
  if (item >= nch * f.tpad * ncw) return;
  if (t >= f.batch) {
    if (f.ncons > 0) zero_chunk(c, t, f.cons[k].fv, f.tpad, f.nj);
    return;
  }
  const bool store = k == 0;
  float yr[2][4];  // the output as stored (what a later reader of y sees), 0 past the rows
  unsigned bad = 0;
  float vs[2][4];
  sum_splits4x2(f.part, f.splits, f.part_stride, (int64_t)t * f.ldp, c * kChunkCols + 4 * lane,
                c * kChunkCols + 4 * (lane + 32), f.rows, vs[0], vs[1]);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j0 = c * kChunkCols + 4 * (lane + 32 * h);
    const bool full = j0 + 3 < f.rows;
    const float (&v)[4] = vs[h];
    float w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      w[e] = v[e] * osc[h][e];
      if (j0 + e < f.rows && !isfinite(w[e])) bad |= kStatusNonFinite;
    }
    const int64_t o = (int64_t)t * f.ldy + j0;
    if (f.y_dtype == DBF_F16) {
      __half hv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hv[e] = __float2half_rn(w[e]);
        if (j0 + e < f.rows && isfinite(w[e]) && __hisinf(hv[e])) bad |= kStatusOverflow;
        yr[h][e] = j0 + e < f.rows ? __half2float(hv[e]) : 0.f;
      }
      if (store) {
        __half* yp = (__half*)f.y + o;
        if (full && ((uintptr_t)yp & 7) == 0) {
          uint2 pk;
          pk.x = (uint32_t)__half_as_ushort(hv[0]) | ((uint32_t)__half_as_ushort(hv[1]) << 16);
          pk.y = (uint32_t)__half_as_ushort(hv[2]) | ((uint32_t)__half_as_ushort(hv[3]) << 16);
          *(uint2*)yp = pk;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (j0 + e < f.rows) yp[e] = hv[e];
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = j0 + e;
        yr[h][e] = 0.f;
        if (j >= f.rows) continue;
        switch (f.y_dtype) {
          case DBF_F32:
            if (store) ((float*)f.y)[o + e] = w[e];
            yr[h][e] = w[e];
            break;
          case DBF_F64:
            if (store) ((double*)f.y)[o + e] = (double)w[e];
            yr[h][e] = w[e];
            break;
          default: {
            const __nv_bfloat16 bv = __float2bfloat16_rn(w[e]);
            if (store) ((__nv_bfloat16*)f.y)[o + e] = bv;
            yr[h][e] = __bfloat162float(bv);
            break;
          }
        }
      }
    }
  }
  if (store) {
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0 && f.status) atomicOr(f.status, bad);
  }
  BT_MARK(f.tslot)
  if (f.ncons == 0) {
    BT_END(f.tslot)
    return;
  }
  float u[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 4; ++e) u[h][e] = yr[h][e] * csc[h][e];
  emit_chunk(u, c, t, f.cons[k].fv, f.tpad, f.nj);
  BT_END(f.tslot)
}

// ---- host side ---------------------------------------------------------------------------------
inline int tpad_of(int64_t batch) { return (int)ceil_div(batch, 4) * 4; }
inline int ldp_of(int64_t rows) { return (int)ceil_div(rows, 4) * 4; }
inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// row blocks per warp: two where there are enough rows (the chunk's B fragments, barriers and
// scale loads then serve twice the MMAs)
// (one above 16 tokens: registers)
inline int rb_per_warp(int64_t nrb, int nj) { return nrb >= 128 && nj <= 4 ? 2 : 1; }
// K splits of one GEMV: enough CTAs for kCtasPerSm per SM, whole chunks per split
inline int split_count(int64_t nrb, int64_t nch, int nj, int* cps) {
  const int64_t gx = ceil_div(nrb, (int64_t)kGemvWarps * rb_per_warp(nrb, nj));
  int64_t S = std::max<int64_t>(1, ceil_div((int64_t)kCtasPerSm * kNumSMs, gx));
  S = std::min<int64_t>(std::min<int64_t>(S, kMaxSplits), nch);
  const int64_t c = ceil_div(nch, S);
  *cps = (int)c;
  return (int)ceil_div(nch, c);
}

// Workspace of one layer: the second GEMV's input fragments, both partial sets, and (for
// dbf_forward_batched, which quantizes x itself) the first GEMV's input fragments
struct Layout {
  size_t frag2, part, frag1, total_frag, total;
};
inline Layout layout_of(int64_t n, int64_t k, int64_t m, int64_t batch) {
  const int tpad = tpad_of(batch);
  int cps;
  const int S1 = split_count(row_blocks(k), chunks(m), tpad / 4, &cps),
            S2 = split_count(row_blocks(n), chunks(k), tpad / 4, &cps);
  Layout L;
  L.frag2 = 0;
  L.part = align256(L.frag2 + frag_bytes(k, tpad));
  // stage-1 partials stay live while stage 2 quantizes from them: both sets side by side
  L.total_frag = align256(L.part + ((size_t)S1 * tpad * ldp_of(k) + (size_t)S2 * tpad * ldp_of(n)) * 4 + 256);
  L.frag1 = L.total_frag;
  L.total = align256(L.frag1 + frag_bytes(m, tpad));
  return L;
}

// diagnostics: the next trace slot (DBF_BATCHED_TRACE builds; -1 otherwise) and the kernel kind
// recorded in column 0 of the slot (1 quantize, 2 gemv, 3 finalize)
#ifdef DBF_BATCHED_TRACE
static int g_next_slot = 0;
static int g_slot_kind[8192];
inline int next_slot(int kind) {
  const int s = g_next_slot < 8192 ? g_next_slot++ : -1;
  if (s >= 0) g_slot_kind[s] = kind;
  return s;
}
#else
inline int next_slot(int) { return -1; }
#endif

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
    case 4: return launch_pdl(gemv_kernel<4, RB>, grid, kGemvWarps * 32, s, a);
    default:
      if constexpr (RB == 1) {
        switch (nj) {
          case 5: return launch_pdl(gemv_kernel<5, 1>, grid, kGemvWarps * 32, s, a);
          case 6: return launch_pdl(gemv_kernel<6, 1>, grid, kGemvWarps * 32, s, a);
          case 7: return launch_pdl(gemv_kernel<7, 1>, grid, kGemvWarps * 32, s, a);
          default: return launch_pdl(gemv_kernel<8, 1>, grid, kGemvWarps * 32, s, a);
        }
      }
      return DBF_ERR_UNSUPPORTED;
  }
}
static int gemv(const GemvArgs& a, int nj, int splits, cudaStream_t s) {
  return rb_per_warp(a.nrb, nj) == 2 ? gemv_rb<2>(a, nj, splits, s) : gemv_rb<1>(a, nj, splits, s);
}

}  // namespace batched
}  // namespace dbf

using namespace dbf;

extern "C" {

size_t dbf_forward_batched_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch) {
  if (n < 1 || k < 1 || m < 1 || batch < 1 || batch > batched::kMaxTokens) return 0;
  return batched::layout_of(n, k, m, batch).total;
}

size_t dbf_batched_frag_bytes(int64_t cols, int64_t batch) {
  if (cols < 1 || batch < 1 || batch > batched::kMaxTokens) return 0;
  return batched::frag_bytes(cols, batched::tpad_of(batch));
}

int dbf_batched_quantize(const void* X, int x_dtype, int64_t ldx, int64_t batch, int64_t cols, const void* iscale,
                         int scale_dtype, void* frag, void* stream) {
  using namespace batched;
  if (!X || !frag || batch < 1 || cols < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (batch > kMaxTokens || cols > INT32_MAX / 2) return DBF_ERR_UNSUPPORTED;
  if (ldx < cols) return DBF_ERR_SHAPE;
  if (!valid_float_dtype(x_dtype) || !valid_float_dtype(scale_dtype)) return DBF_ERR_INVALID_ARGUMENT;
  const int tpad = tpad_of(batch);
  QuantIn q{};
  q.x = X, q.x_dtype = x_dtype, q.ldx = ldx, q.iscale = iscale, q.scale_dtype = scale_dtype;
  q.cols = (int)cols, q.batch = (int)batch, q.tpad = tpad, q.tslot = next_slot(1);
  return launch_pdl(quantize_kernel, dim3((unsigned)ceil_div(chunks(cols) * tpad, kWarps)), kThreads,
                    (cudaStream_t)stream, q, frag_view(frag, cols, tpad), tpad / 4);
}

size_t dbf_forward_batched_frag_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch) {
  if (n < 1 || k < 1 || m < 1 || batch < 1 || batch > batched::kMaxTokens) return 0;
  return batched::layout_of(n, k, m, batch).total_frag;
}

int dbf_forward_batched_frag(const void* A_tiled, const void* B_tiled, const void* a, const void* mid,
                             int scale_dtype, int64_t n, int64_t k, int64_t m, const void* frag_in, int64_t batch,
                             void* Y, int y_dtype, int64_t ldy, const dbf_batched_consumer* consumers,
                             int nconsumers, void* workspace, size_t workspace_bytes, unsigned* status,
                             void* stream) {
  using namespace batched;
  if (!A_tiled || !B_tiled || !frag_in || !Y) return DBF_ERR_INVALID_ARGUMENT;
  if (n < 1 || k < 1 || m < 1 || batch < 1 || nconsumers < 0) return DBF_ERR_INVALID_ARGUMENT;
  if (nconsumers > 0 && !consumers) return DBF_ERR_INVALID_ARGUMENT;
  if (batch > kMaxTokens || nconsumers > kMaxConsumers) return DBF_ERR_UNSUPPORTED;
  if (n > INT32_MAX / 2 || k > INT32_MAX / 2 || m > INT32_MAX / 2) return DBF_ERR_UNSUPPORTED;
  if (ldy < n) return DBF_ERR_SHAPE;
  if (!valid_float_dtype(y_dtype) || !valid_float_dtype(scale_dtype)) return DBF_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < nconsumers; ++i)
    if (!consumers[i].frag) return DBF_ERR_INVALID_ARGUMENT;
  const Layout L = layout_of(n, k, m, batch);
  if (!workspace || workspace_bytes < L.total_frag) return DBF_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  const int tpad = tpad_of(batch), nj = tpad / 4;
  int cps1, cps2;
  const int S1 = split_count(row_blocks(k), chunks(m), nj, &cps1), S2 = split_count(row_blocks(n), chunks(k), nj, &cps2);
  const int ldk = ldp_of(k), ldn = ldp_of(n);
  float* part1 = (float*)(ws + L.part);
  float* part2 = part1 + (size_t)S1 * tpad * ldk;
  const FragView f1 = frag_view(const_cast<void*>(frag_in), m, tpad), f2 = frag_view(ws + L.frag2, k, tpad);

  // t = mid * (B . (x * b))
  GemvArgs g1{(const uint4*)B_tiled, (int)k, (int)row_blocks(k), (int)chunks(m), cps1, f1.bfrag, f1.F, f1.T, tpad,
              (int)batch, part1, ldk, next_slot(2)};
  int st = gemv(g1, nj, S1, s);
  if (st != DBF_OK) return st;
  // t quantized straight from the stage-1 partials
  QuantIn q2{};
  q2.part = part1, q2.splits = S1, q2.ldx = ldk, q2.part_stride = (int64_t)tpad * ldk, q2.pscale = mid;
  q2.scale_dtype = scale_dtype, q2.cols = (int)k, q2.batch = (int)batch, q2.tpad = tpad, q2.tslot = next_slot(1);
  st = launch_pdl(quantize_kernel, dim3((unsigned)ceil_div(chunks(k) * tpad, kWarps)), kThreads, s, q2, f2, nj);
  if (st != DBF_OK) return st;
  // y = a * (A . t)
  GemvArgs g2{(const uint4*)A_tiled, (int)n, (int)row_blocks(n), (int)chunks(k), cps2, f2.bfrag, f2.F, f2.T, tpad,
              (int)batch, part2, ldn, next_slot(2)};
  if ((st = gemv(g2, nj, S2, s)) != DBF_OK) return st;
  FinArgs fa{};
  fa.part = part2, fa.splits = S2, fa.part_stride = (int64_t)tpad * ldn, fa.ldp = ldn, fa.rows = (int)n;
  fa.batch = (int)batch, fa.tpad = tpad, fa.nj = nj, fa.oscale = a, fa.scale_dtype = scale_dtype;
  fa.y = Y, fa.y_dtype = y_dtype, fa.ldy = ldy, fa.status = status, fa.ncons = nconsumers, fa.tslot = next_slot(3);
  for (int i = 0; i < nconsumers; ++i) fa.cons[i] = Consumer{consumers[i].b, frag_view(consumers[i].frag, n, tpad)};
  return launch_pdl(finalize_kernel, dim3((unsigned)ceil_div(chunks(n) * tpad * std::max(1, nconsumers), kWarps)),
                    kThreads, s, fa);
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
  const Layout L = layout_of(n, k, m, batch);
  if (!workspace || workspace_bytes < L.total) return DBF_ERR_WORKSPACE;
  void* frag1 = (char*)workspace + L.frag1;
  const int st = dbf_batched_quantize(X, x_dtype, ldx, batch, m, b, scale_dtype, frag1, stream);
  if (st != DBF_OK) return st;
  return dbf_forward_batched_frag(A_tiled, B_tiled, a, mid, scale_dtype, n, k, m, frag1, batch, Y, y_dtype, ldy,
                                  nullptr, 0, workspace, L.total_frag, status, stream);
}

// diagnostics (DBF_BATCHED_TRACE builds; DBF_ERR_UNSUPPORTED otherwise): reset every trace slot /
// restart slot numbering, and copy n slots (kind, first CTA start, last grid_wait exit, last end)
int dbf_batched_debug_reset(int restart_slots) {
#ifdef DBF_BATCHED_TRACE
  static unsigned long long init[8192][5];
  for (int i = 0; i < 8192; ++i) init[i][0] = 0, init[i][1] = ~0ull, init[i][2] = 0, init[i][3] = 0, init[i][4] = 0;
  if (restart_slots) batched::g_next_slot = 0;
  return cudaMemcpyToSymbol(batched::g_btrace, init, sizeof(init)) == cudaSuccess ? DBF_OK : DBF_ERR_CUDA;
#else
  (void)restart_slots;
  return DBF_ERR_UNSUPPORTED;
#endif
}
int dbf_batched_debug_trace(unsigned long long* host, int n) {
#ifdef DBF_BATCHED_TRACE
  if (n > 8192) n = 8192;
  if (cudaMemcpyFromSymbol(host, batched::g_btrace, (size_t)n * 40) != cudaSuccess) return DBF_ERR_CUDA;
  for (int i = 0; i < n; ++i) host[5 * i] = (unsigned long long)batched::g_slot_kind[i];
  return DBF_OK;
#else
  (void)host, (void)n;
  return DBF_ERR_UNSUPPORTED;
#endif
}

}  // extern "C"
