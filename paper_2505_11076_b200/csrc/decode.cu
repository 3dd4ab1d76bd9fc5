// Decode path of the DBF forward on B200: the tensor-core sign GEMV.
//
// Replaces kernel.sign_matvec / kernel.forward (/root/reference/pkg/src/dbf/kernel.py:24-62).
// The reference accumulates pos - neg sums in float64 over 64-column words; here
//
//   (1) each input row u = x * iscale is quantized ONCE to a 22-bit fixed-point grid relative
//       to its max |u|:  X_j = rint(u_j * 2^F),  F = 22 - exponent(max|u|)  (exact scaling);
//   (2) the sign product is split as  sum_j s_j X_j = 2 * sum_{bit_j=1} X_j - sum_j X_j;
//   (3) sum_{bit=1} X_j runs on the int8 tensor cores (mma.sync m16n8k32 u8 x s8 -> s32, the
//       native IMMA.16832 on sm_100a).  The A operand is the packed sign word ANDed with
//       0x01010101 << r, i.e. the value 2^r * bit -- one LOP3 per four weights, no shifts.  The
//       B operand holds the balanced base-256 digits of X_j * 2^(7 - r), so every product is
//       2^7 * bit_j * X_j whatever the bit position r;
//   (4) the int32 accumulators are recombined exactly in int64 and scaled once per output.
//
// All arithmetic after the quantization is exact integer arithmetic, so results are bitwise
// reproducible (test_kernel.py:47-50) and independent of the reduction order.
#include <algorithm>
#include "common.cuh"

namespace dbf {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kBadF = -(1 << 20);  // exponent marking a row that held inf / NaN
constexpr int kQuantBits = 22;  // |X| <= 2^22; X * 2^7 fits 4 balanced int8 digits with room

struct GemvParams {
  const uint4* tiled;  // tiled sign matrix (dbf_tile_signs)
  int rows, cols;      // logical shape
  int nrb, nchunks;    // 16-row blocks, 256-column chunks
  const void* x;       // input rows (x_dtype), row stride ldx elements
  int64_t ldx;
  int x_dtype;
  int batch;           // rows of x handled by this launch
  const void* iscale;  // per-column input scale (scale_dtype) or null
  const void* oscale;  // per-row output scale (scale_dtype) or null
  int scale_dtype;
  void* y;             // output rows (y_dtype), row stride ldy
  int64_t ldy;
  int y_dtype;
  // fused one-shot all-reduce (k-sharded GEMV2, dbf_forward_allreduce); ar_world == 0 = off
  int ar_world, ar_rank, ar_group, ar_bt, ar_row0;
  const uint32_t* ar_epoch;  // device call counter (GEMV2 reads it)
  uint32_t* bump;            // GEMV1's first launch advances the counter (block 0, thread 0)
  const uint64_t* ar_recv;   // [world] peer receive buffers, each [2][world][ar_bt][rows] fp32
  const uint64_t* ar_flags;  // [world] peer flag arrays, each [kArGroups][world][nrb] u32
  const void* ar_a;          // output scale a (scale_dtype)
  void* ar_y;                // final output (ar_ydt), row stride ar_ldy
  int64_t ar_ldy;
  int ar_ydt;
};

constexpr int kArGroups = 16;  // launches per call that may share the flag array (batch <= 32)

__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double load_any(const void* p, int dt, int64_t i) {
  switch (dt) {
    case DBF_F16: return (double)__half2float(((const __half*)p)[i]);
    case DBF_F32: return (double)((const float*)p)[i];
    case DBF_F64: return ((const double*)p)[i];
    default: return (double)__bfloat162float(((const __nv_bfloat16*)p)[i]);
  }
}
__device__ __forceinline__ float load_any_f(const void* p, int dt, int64_t i) {
  switch (dt) {
    case DBF_F16: return __half2float(((const __half*)p)[i]);
    case DBF_F32: return ((const float*)p)[i];
    case DBF_F64: return (float)((const double*)p)[i];
    default: return __bfloat162float(((const __nv_bfloat16*)p)[i]);
  }
}
__device__ __forceinline__ void store_any(void* p, int dt, int64_t i, double v) {
  switch (dt) {
    case DBF_F16: ((__half*)p)[i] = __float2half_rn((float)v); break;
    case DBF_F32: ((float*)p)[i] = (float)v; break;
    case DBF_F64: ((double*)p)[i] = v; break;
    default: ((__nv_bfloat16*)p)[i] = __float2bfloat16_rn((float)v); break;
  }
}

__device__ __forceinline__ void imma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// exponent e with v = mant * 2^e, mant in [0.5, 1)  (v > 0, finite)
__device__ __forceinline__ int frexp_exp(double v) { int e; frexp(v, &e); return e; }

// 2^F as a double (exact for the F range reachable from finite inputs).
__device__ __forceinline__ double pow2(int F) { return ldexp(1.0, F); }

// Four balanced int8 digits of v (|v| < 2^31 - 2^23): bytes of (v + 0x808080) ^ 0x808080.
__device__ __forceinline__ uint32_t digits4(int32_t v) {
  return ((uint32_t)v + 0x00808080u) ^ 0x00808080u;
}

// Quantize one input row into the B-fragment layout.
//   xfrag[(pair * nkb + kb) * lpk + lane][8 bytes]:  lane = 16*bsub + 4*plane + tig,
//   bytes 0..3 -> k = 4*tig + 0..3 of k-block kb, bytes 4..7 -> k = 16 + 4*tig + 0..3.
// Returns (via smem) F and T = sum_j X_j for the row.
template <typename AT>
__device__ void quantize_row(const GemvParams& p, int slot, int nkb, int lpk, uint8_t* xfrag,
                             int* sF, long long* sT, AT* red_max, long long* red_sum) {
  const int tid = threadIdx.x;
  const void* xr = (const char*)p.x + (int64_t)slot * p.ldx * (int64_t)(p.x_dtype == DBF_F64 ? 8 : (p.x_dtype == DBF_F32 ? 4 : 2));
  // pass 1: max |x * iscale|
  AT mx = 0;
  int nonfinite = 0;
  for (int j = tid; j < p.cols; j += kThreads) {
    AT u = (AT)load_any(xr, p.x_dtype, j);
    if (p.iscale) u *= (AT)load_any(p.iscale, p.scale_dtype, j);
    mx = fmax(mx, fabs(u));
    nonfinite |= !isfinite((double)u);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red_max[tid >> 5] = mx;
  __syncthreads();
  if (tid == 0) {
    AT m = 0;
    for (int w = 0; w < kWarps; ++w) m = fmax(m, red_max[w]);
    // an inf max: F = kBadF (zero digits, NaN outputs); a NaN is caught by the vote below
    int F = (m > 0) ? kQuantBits - frexp_exp((double)m) : 0;
    if (!isfinite((double)m)) F = kBadF;
    *sF = F;
  }
  __syncthreads();
  // any NaN in the row (fmax drops NaN operands, so the max alone cannot see it)
  if (__syncthreads_or(nonfinite)) {
    if (tid == 0) *sF = kBadF;
  }
  __syncthreads();
  const int F = *sF;
  const AT scale = F == kBadF ? (AT)0 : (AT)pow2(F);
  // pass 2: groups of 4 consecutive columns -> 4 digit planes of 4 bytes each
  const int pair = slot >> 1, bsub = slot & 1;
  const int ngroups = nkb * 8;
  long long tsum = 0;
  for (int q = tid; q < ngroups; q += kThreads) {
    const int kb = q >> 3, r = kb & 7, tig = q & 3, half = (q >> 2) & 1;
    uint32_t d[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = q * 4 + e;
      int32_t X = 0;
      if (j < p.cols) {
        AT u = (AT)load_any(xr, p.x_dtype, j);
        if (p.iscale) u *= (AT)load_any(p.iscale, p.scale_dtype, j);
        X = (int32_t)rint(u * scale);
      }
      tsum += X;
      d[e] = digits4(X * (1 << (7 - r)));
    }
    // byte transpose: plane k word = byte k of d[0..3]
    const uint32_t t0 = __byte_perm(d[0], d[1], 0x5140), t1 = __byte_perm(d[0], d[1], 0x7362);
    const uint32_t t2 = __byte_perm(d[2], d[3], 0x5140), t3 = __byte_perm(d[2], d[3], 0x7362);
    const uint32_t P0 = __byte_perm(t0, t2, 0x5410), P1 = __byte_perm(t0, t2, 0x7632);
    const uint32_t P2 = __byte_perm(t1, t3, 0x5410), P3 = __byte_perm(t1, t3, 0x7632);
    uint8_t* base = xfrag + ((int64_t)(pair * nkb + kb) * lpk) * 8 + 4 * half;
    const int l0 = 16 * bsub + tig;
    *(uint32_t*)(base + (l0 + 0) * 8) = P0;
    *(uint32_t*)(base + (l0 + 4) * 8) = P1;
    *(uint32_t*)(base + (l0 + 8) * 8) = P2;
    *(uint32_t*)(base + (l0 + 12) * 8) = P3;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
  if ((tid & 31) == 0) red_sum[tid >> 5] = tsum;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int w = 0; w < kWarps; ++w) t += red_sum[w];
    *sT = t;
  }
  __syncthreads();
}

// Batched launches quantize every input row ONCE (one CTA per row, fragments written to the
// workspace in the B-fragment layout with lpk = 32) instead of once per GEMV CTA; the GEMV CTAs
// then only copy the fragments of their row pairs into shared memory (PRE = true).
template <typename AT>
__global__ void __launch_bounds__(kThreads) quantize_rows_kernel(GemvParams p, int batch_total, int nkb,
                                                                 uint8_t* gfrag, int* gF, long long* gT) {
  __shared__ AT red_max[kWarps];
  __shared__ long long red_sum[kWarps];
  __shared__ int sF;
  __shared__ long long sT;
  const int slot = blockIdx.x;
  if (slot < batch_total) {
    quantize_row<AT>(p, slot, nkb, 32, gfrag, &sF, &sT, red_max, red_sum);
    if (threadIdx.x == 0) { gF[slot] = sF; gT[slot] = sT; }
  } else {  // zero half of the last pair
    const int pair = slot >> 1, bsub = slot & 1;
    for (int q = threadIdx.x; q < nkb * 16; q += kThreads) {
      const int kb = q >> 4, rem = q & 15;
      *(uint2*)(gfrag + ((int64_t)(pair * nkb + kb) * 32 + 16 * bsub + rem) * 8) = make_uint2(0, 0);
    }
    if (threadIdx.x == 0) { gF[slot] = 0; gT[slot] = 0; }
  }
}

// One CTA = 8 warps; a 16-row block is split across warps by 256-column chunks.
// NP = pairs of input rows per launch (B-fragment columns n = 4*bsub + plane).
// SINGLE = one input row: only lanes 0..15 carry B fragments (lanes 16..31 feed zeros).
template <int NP, bool SINGLE, bool PRE>
__global__ void __launch_bounds__(kThreads) gemv_i8_kernel(GemvParams p, const uint8_t* gfrag, const int* gF,
                                                          const long long* gT) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int nkb = p.nchunks * 8;
  constexpr int lpk = SINGLE ? 16 : 32;
  uint8_t* xfrag = smem;
  const size_t xfrag_bytes = (size_t)NP * nkb * lpk * 8;
  long long* red = (long long*)(smem + xfrag_bytes);            // [kWarps][16][2*NP]
  long long* sT = red + kWarps * 16 * 2 * NP;                    // [2*NP]
  int* sF = (int*)(sT + 2 * NP);                                 // [2*NP]
  double* red_max = (double*)(sF + 2 * NP + 2);                  // [kWarps] (8-byte aligned)
  long long* red_sum = (long long*)(red_max + kWarps);           // [kWarps]

  // ---- prologue: B fragments of every input row of this launch into shared memory
  const int slots = SINGLE ? 1 : 2 * NP;
  if constexpr (PRE) {  // pre-quantized by quantize_rows_kernel: a straight copy
    const uint4* src = (const uint4*)gfrag;
    uint4* dst = (uint4*)xfrag;
    const int n16 = (int)(xfrag_bytes / 16);
    for (int i = threadIdx.x; i < n16; i += kThreads) dst[i] = __ldg(src + i);
    if (threadIdx.x < slots) {
      sF[threadIdx.x] = gF[threadIdx.x];
      sT[threadIdx.x] = gT[threadIdx.x];
    }
  } else for (int s = 0; s < slots; ++s) {
    if (s < p.batch) {
      if (p.x_dtype == DBF_F64)
        quantize_row<double>(p, s, nkb, lpk, xfrag, sF + s, sT + s, red_max, red_sum);
      else
        quantize_row<float>(p, s, nkb, lpk, xfrag, sF + s, sT + s, (float*)red_max, red_sum);
    } else {
      // zero-fill the unused half of the last pair
      const int pair = s >> 1, bsub = s & 1;
      for (int q = threadIdx.x; q < nkb * 16; q += kThreads) {
        const int kb = q >> 4, rem = q & 15;  // rem -> (plane, tig)
        *(uint2*)(xfrag + ((int64_t)(pair * nkb + kb) * lpk + 16 * bsub + rem) * 8) = make_uint2(0, 0);
      }
      if (threadIdx.x == 0) { sF[s] = 0; sT[s] = 0; }
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const uint2* xf2 = (const uint2*)xfrag;
  if (p.bump && blockIdx.x == 0 && threadIdx.x == 0) *p.bump += 1u;
  const uint32_t ar_epoch = p.ar_world ? *(const volatile uint32_t*)p.ar_epoch : 0u;

  for (int rb = blockIdx.x; rb < p.nrb; rb += gridDim.x) {
    int acc[NP][4];
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0;

    const uint4* wbase = p.tiled + (int64_t)rb * p.nchunks * 32 + lane;
    int c = warp;
    uint4 w = (c < p.nchunks) ? __ldg(wbase + c * 32) : make_uint4(0, 0, 0, 0);
    for (; c < p.nchunks; c += kWarps) {
      const int cn = c + kWarps;
      const uint4 wn = (cn < p.nchunks) ? __ldg(wbase + cn * 32) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint32_t m = 0x01010101u << r;
        const uint32_t a0 = w.x & m, a1 = w.y & m, a2 = w.z & m, a3 = w.w & m;
        const int kb = c * 8 + r;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          uint2 b = make_uint2(0, 0);
          if (!SINGLE || lane < 16) b = xf2[(q * nkb + kb) * lpk + lane];
          imma_u8s8(acc[q], a0, a1, a2, a3, b.x, b.y);
        }
      }
      w = wn;
    }
    // ---- combine digit planes: columns n = 2*tig, 2*tig+1 -> (bsub = tig>>1, planes 2*(tig&1)+{0,1})
    const int sh = 16 * (tig & 1);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      long long v0 = (long long)acc[q][0] * (1LL << sh) + (long long)acc[q][1] * (1LL << (sh + 8));
      long long v1 = (long long)acc[q][2] * (1LL << sh) + (long long)acc[q][3] * (1LL << (sh + 8));
      v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
      v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
      if ((tig & 1) == 0) {
        const int slot = 2 * q + (tig >> 1);
        red[(warp * 16 + g) * 2 * NP + slot] = v0;
        red[(warp * 16 + g + 8) * 2 * NP + slot] = v1;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * slots; t += kThreads) {
      const int row = t & 15, slot = t >> 4;
      const int grow = rb * 16 + row;
      if (slot < p.batch && grow < p.rows) {
        long long s128 = 0;
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) s128 += red[(w2 * 16 + row) * 2 * NP + slot];
        const long long P = 2 * (s128 >> 7) - sT[slot];
        // a row with a non-finite input (F = kBadF, zero digits) gives NaN, never a finite value
        double v = sF[slot] == kBadF ? __longlong_as_double(0x7FF8000000000000ll) : (double)P * pow2(-sF[slot]);
        if (p.oscale) v *= load_any(p.oscale, p.scale_dtype, grow);
        if (p.ar_world == 1) {
          // world 1: nothing to exchange -- the combine's formula applied in place (same bits as
          // the push / flag / combine path, without its system-scope fence and flag round trip)
          store_any(p.ar_y, p.ar_ydt, (int64_t)(p.ar_row0 + slot) * p.ar_ldy + grow,
                    (double)(float)v * load_any(p.ar_a, p.scale_dtype, grow));
        } else if (p.ar_world) {
          // one-shot all-reduce, push half: this rank's fp32 partial into slot `ar_rank` of every
          // peer's receive buffer (NVLink P2P stores through the peers' mapped addresses)
          const float fv = (float)v;
          const size_t idx = (size_t)(ar_epoch & 1u) * p.ar_world * p.ar_bt * p.rows +
                             ((size_t)p.ar_rank * p.ar_bt + p.ar_row0 + slot) * p.rows + grow;
          for (int g2 = 0; g2 < p.ar_world; ++g2) ((float*)p.ar_recv[g2])[idx] = fv;
        } else {
          store_any(p.y, p.y_dtype, (int64_t)slot * p.ldy + grow, v);
        }
      }
    }
    __syncthreads();
  }
  if (p.ar_world <= 1) return;
  // this CTA's row blocks are out: ONE system-scope fence, then release them to every peer
  // (flag = epoch, monotonic); a fence per row block cost more than the GEMV itself
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int rb = blockIdx.x; rb < p.nrb; rb += gridDim.x)
      for (int g2 = 0; g2 < p.ar_world; ++g2)
        st_relaxed_sys((uint32_t*)p.ar_flags[g2] + ((size_t)p.ar_group * p.ar_world + p.ar_rank) * p.nrb + rb,
                       ar_epoch);
  }
  // ---- one-shot all-reduce, combine half: wait until every rank has pushed every row block this
  // CTA produced (all flags polled in parallel), then y = a * sum over ranks in rank order
  // (identical bits on every rank)
  const uint32_t* myflags = (const uint32_t*)p.ar_flags[p.ar_rank] + (size_t)p.ar_group * p.ar_world * p.nrb;
  const float* recv = (const float*)p.ar_recv[p.ar_rank] + (size_t)(ar_epoch & 1u) * p.ar_world * p.ar_bt * p.rows;
  const int nmy = (p.nrb - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  for (int i = threadIdx.x; i < nmy * p.ar_world; i += kThreads) {
    const int rb = blockIdx.x + (i / p.ar_world) * gridDim.x, src = i % p.ar_world;
    const uint32_t* f = myflags + (size_t)src * p.nrb + rb;
    const uint64_t t0 = global_ns();
    // epochs only grow: a peer already on the next call has also pushed this one
    while ((int32_t)(ld_acquire_sys(f) - ar_epoch) < 0) {
      __nanosleep(64);
      if (global_ns() - t0 > 20ull * 1000 * 1000 * 1000) __trap();  // 20 s watchdog: a peer is gone
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nmy * 16 * slots; i += kThreads) {
    const int t = i % (16 * slots), row = t & 15, slot = t >> 4;
    const int grow = (blockIdx.x + (i / (16 * slots)) * gridDim.x) * 16 + row;
    if (slot < p.batch && grow < p.rows) {
      double acc = 0.0;
      for (int src = 0; src < p.ar_world; ++src)
        acc += (double)__ldcg(recv + ((size_t)src * p.ar_bt + p.ar_row0 + slot) * p.rows + grow);
      store_any(p.ar_y, p.ar_ydt, (int64_t)(p.ar_row0 + slot) * p.ar_ldy + grow,
                (double)(float)acc * load_any(p.ar_a, p.scale_dtype, grow));
    }
  }
}

size_t gemv_smem_bytes(int np, bool single, int nchunks) {
  const int nkb = nchunks * 8;
  const int lpk = single ? 16 : 32;
  return (size_t)np * nkb * lpk * 8 + (size_t)kWarps * 16 * 2 * np * 8 + 2 * np * 8 +
         (2 * np + 2) * 4 + kWarps * 8 + kWarps * 8 + 16;
}

template <int NP, bool SINGLE, bool PRE = false>
int launch_gemv_t(const GemvParams& p, cudaStream_t s, const uint8_t* gfrag = nullptr, const int* gF = nullptr,
                  const long long* gT = nullptr) {
  const size_t smem = gemv_smem_bytes(NP, SINGLE, p.nchunks);
  const int st = ensure_smem_attr<gemv_i8_kernel<NP, SINGLE, PRE>>(227 * 1024);
  if (st != DBF_OK) return st;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_i8_kernel<NP, SINGLE, PRE>, kThreads, smem);
  per_sm = std::max(per_sm, 1);
  const int grid = std::min<int64_t>(p.nrb, (int64_t)kNumSMs * per_sm);
  gemv_i8_kernel<NP, SINGLE, PRE><<<grid, kThreads, smem, s>>>(p, gfrag, gF, gT);
  return check_launch();
}

constexpr size_t kMaxSmem = 227 * 1024;

// Workspace for pre-quantized fragments of `batch` rows of `cols` columns (lpk = 32 layout).
size_t frag_bytes(int64_t cols, int64_t batch) {
  const int64_t pairs = (batch + 1) / 2;
  return (size_t)pairs * chunks(cols) * 8 * 32 * 8 + (size_t)(2 * pairs) * (4 + 8) + 64;
}

// Batched rows (>= 2): quantize once into `ws` (frag_bytes), then one GEMV launch per group of up
// to 8 row pairs copying its fragments.
int run_gemv_pre(GemvParams p, int batch_total, cudaStream_t s, uint8_t* ws) {
  const int nkb = p.nchunks * 8;
  const int64_t pairs = (batch_total + 1) / 2;
  uint8_t* gfrag = ws;
  long long* gT = (long long*)(ws + (size_t)pairs * nkb * 32 * 8);
  int* gF = (int*)(gT + 2 * pairs);
  const int qgrid = (int)(2 * pairs);
  if (p.x_dtype == DBF_F64)
    quantize_rows_kernel<double><<<qgrid, kThreads, 0, s>>>(p, batch_total, nkb, gfrag, gF, gT);
  else
    quantize_rows_kernel<float><<<qgrid, kThreads, 0, s>>>(p, batch_total, nkb, gfrag, gF, gT);
  int st = check_launch();
  if (st != DBF_OK) return st;
  const size_t ysz = dtype_size(p.y_dtype);
  int done = 0;  // rows
  int group = 0;
  while (done < batch_total) {
    const int left = batch_total - done;
    int np = 8;
    while (np > 1 && (2 * np > left + 1 || gemv_smem_bytes(np, false, p.nchunks) > 227 * 1024)) np >>= 1;
    if (gemv_smem_bytes(np, false, p.nchunks) > 227 * 1024) return DBF_ERR_UNSUPPORTED;
    const int take = std::min(left, 2 * np);
    GemvParams q = p;
    q.y = (char*)p.y + (int64_t)done * p.ldy * ysz;
    q.batch = take;
    if (done > 0) q.bump = nullptr;
    if (q.ar_world) {
      q.ar_row0 = done;
      q.ar_group = group++;
      if (q.ar_group >= kArGroups) return DBF_ERR_UNSUPPORTED;
    }
    const int pair0 = done / 2;
    const uint8_t* f = gfrag + (size_t)pair0 * nkb * 32 * 8;
    switch (np) {
      case 8: st = launch_gemv_t<8, false, true>(q, s, f, gF + done, gT + done); break;
      case 4: st = launch_gemv_t<4, false, true>(q, s, f, gF + done, gT + done); break;
      case 2: st = launch_gemv_t<2, false, true>(q, s, f, gF + done, gT + done); break;
      default: st = launch_gemv_t<1, false, true>(q, s, f, gF + done, gT + done); break;
    }
    if (st != DBF_OK) return st;
    done += take;
  }
  return DBF_OK;
}

// Runs the GEMV for all `batch` rows, grouping rows so that the B fragments fit in smem.
int run_gemv(GemvParams p, int batch_total, cudaStream_t s, uint8_t* ws = nullptr, size_t ws_bytes = 0) {
  if (batch_total >= 2 && ws && ws_bytes >= frag_bytes(p.cols, batch_total) &&
      gemv_smem_bytes(1, false, p.nchunks) <= 227 * 1024)
    return run_gemv_pre(p, batch_total, s, ws);
  const size_t xsz = dtype_size(p.x_dtype), ysz = dtype_size(p.y_dtype);
  int done = 0, group = 0;
  while (done < batch_total) {
    const int left = batch_total - done;
    GemvParams q = p;
    q.x = (const char*)p.x + (int64_t)done * p.ldx * xsz;
    q.y = (char*)p.y + (int64_t)done * p.ldy * ysz;
    if (done > 0) q.bump = nullptr;
    if (q.ar_world) {
      q.ar_row0 = done;
      q.ar_group = group++;
      if (q.ar_group >= kArGroups) return DBF_ERR_UNSUPPORTED;
    }
    int st;
    int take;
    if (left == 1 || gemv_smem_bytes(1, false, p.nchunks) > kMaxSmem) {
      if (gemv_smem_bytes(1, true, p.nchunks) > kMaxSmem) return DBF_ERR_UNSUPPORTED;
      take = 1;
      q.batch = 1;
      st = launch_gemv_t<1, true>(q, s);
    } else {
      int np = 8;
      while (np > 1 && (2 * np > left + 1 || gemv_smem_bytes(np, false, p.nchunks) > kMaxSmem)) np >>= 1;
      take = std::min(left, 2 * np);
      q.batch = take;
      switch (np) {
        case 8: st = launch_gemv_t<8, false>(q, s); break;
        case 4: st = launch_gemv_t<4, false>(q, s); break;
        case 2: st = launch_gemv_t<2, false>(q, s); break;
        default: st = launch_gemv_t<1, false>(q, s); break;
      }
    }
    if (st != DBF_OK) return st;
    done += take;
  }
  return DBF_OK;
}

GemvParams make_params(const void* tiled, int64_t rows, int64_t cols, const void* x, int x_dtype,
                       int64_t ldx, const void* iscale, const void* oscale, int scale_dtype,
                       void* y, int y_dtype, int64_t ldy) {
  GemvParams p{};
  p.tiled = (const uint4*)tiled;
  p.rows = (int)rows;
  p.cols = (int)cols;
  p.nrb = (int)row_blocks(rows);
  p.nchunks = (int)chunks(cols);
  p.x = x;
  p.ldx = ldx;
  p.x_dtype = x_dtype;
  p.iscale = iscale;
  p.oscale = oscale;
  p.scale_dtype = scale_dtype;
  p.y = y;
  p.ldy = ldy;
  p.y_dtype = y_dtype;
  return p;
}

inline bool io_dtype_ok(int dt) { return dt == DBF_F16 || dt == DBF_F32 || dt == DBF_F64 || dt == DBF_BF16; }
inline bool scale_dtype_ok(int dt) { return dt == DBF_F16 || dt == DBF_F32 || dt == DBF_F64; }
inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace dbf

using namespace dbf;

extern "C" size_t dbf_forward_workspace_bytes(int64_t n, int64_t k, int64_t m, int64_t batch) {
  (void)n;
  if (k < 1 || batch < 1) return 0;
  // t (fp32) + pre-quantized B fragments for the wider stage input (batches >= 2)
  const size_t frag = batch >= 2 ? frag_bytes(std::max(k, m), batch) : 0;
  return align256((size_t)batch * k * sizeof(float)) + align256(frag);
}

extern "C" int dbf_sign_matvec(const void* S_tiled, int64_t rows, int64_t cols, const void* X,
                               int x_dtype, int64_t batch, int64_t ldx, void* Y, int y_dtype,
                               int64_t ldy, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!S_tiled || !X || !Y || rows < 1 || cols < 1 || batch < 1 || ldx < cols || ldy < rows ||
      !io_dtype_ok(x_dtype) || !io_dtype_ok(y_dtype) || rows > INT32_MAX || cols > INT32_MAX)
    return DBF_ERR_INVALID_ARGUMENT;
  GemvParams p = make_params(S_tiled, rows, cols, X, x_dtype, ldx, nullptr, nullptr, DBF_F32, Y,
                             y_dtype, ldy);
  return run_gemv(p, (int)batch, (cudaStream_t)stream, (uint8_t*)workspace, workspace ? workspace_bytes : 0);
}

extern "C" int dbf_forward(const void* A_tiled, const void* B_tiled, const void* a, const void* mid,
                           const void* b, int scale_dtype, int64_t n, int64_t k, int64_t m,
                           const void* X, int x_dtype, int64_t batch, int64_t ldx, void* Y,
                           int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes,
                           void* stream) {
  if (!A_tiled || !B_tiled || !a || !mid || !b || !X || !Y || n < 1 || k < 1 || m < 1 ||
      batch < 1 || ldx < m || ldy < n || !io_dtype_ok(x_dtype) || !io_dtype_ok(y_dtype) ||
      !scale_dtype_ok(scale_dtype))
    return DBF_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < dbf_forward_workspace_bytes(n, k, m, batch))
    return DBF_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  float* t = (float*)workspace;
  uint8_t* fw = (uint8_t*)workspace + align256((size_t)batch * k * sizeof(float));
  const size_t fwb = workspace_bytes - align256((size_t)batch * k * sizeof(float));
  // stage 1: t = mid * (B . (b * x))      (kernel.py:59 + the `* layer.mid` of kernel.py:60)
  GemvParams p1 = make_params(B_tiled, k, m, X, x_dtype, ldx, b, mid, scale_dtype, t, DBF_F32, k);
  int st = run_gemv(p1, (int)batch, s, fw, fwb);
  if (st != DBF_OK) return st;
  // stage 2: y = a * (A . t)               (kernel.py:60-61)
  GemvParams p2 = make_params(A_tiled, n, k, t, DBF_F32, k, nullptr, a, scale_dtype, Y, y_dtype, ldy);
  return run_gemv(p2, (int)batch, s, fw, fwb);
}

extern "C" int dbf_forward_partial(const void* A_shard_tiled, const void* B_shard_tiled,
                                   const void* mid_shard, const void* b, int scale_dtype, int64_t n,
                                   int64_t k_shard, int64_t m, const void* X, int x_dtype,
                                   int64_t batch, int64_t ldx, float* P, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (!A_shard_tiled || !B_shard_tiled || !mid_shard || !b || !X || !P || n < 1 || k_shard < 1 ||
      m < 1 || batch < 1 || ldx < m || !io_dtype_ok(x_dtype) || !scale_dtype_ok(scale_dtype))
    return DBF_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < dbf_forward_workspace_bytes(n, k_shard, m, batch))
    return DBF_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  float* t = (float*)workspace;
  uint8_t* fw = (uint8_t*)workspace + align256((size_t)batch * k_shard * sizeof(float));
  const size_t fwb = workspace_bytes - align256((size_t)batch * k_shard * sizeof(float));
  GemvParams p1 = make_params(B_shard_tiled, k_shard, m, X, x_dtype, ldx, b, mid_shard, scale_dtype,
                              t, DBF_F32, k_shard);
  int st = run_gemv(p1, (int)batch, s, fw, fwb);
  if (st != DBF_OK) return st;
  GemvParams p2 = make_params(A_shard_tiled, n, k_shard, t, DBF_F32, k_shard, nullptr, nullptr,
                              scale_dtype, P, DBF_F32, n);
  return run_gemv(p2, (int)batch, s, fw, fwb);
}

extern "C" size_t dbf_allreduce_recv_bytes(int64_t n, int64_t batch, int world) {
  if (n < 1 || batch < 1 || world < 1) return 0;
  return (size_t)2 * world * batch * n * sizeof(float);
}

extern "C" size_t dbf_allreduce_flag_bytes(int64_t n, int world) {
  if (n < 1 || world < 1) return 0;
  return (size_t)kArGroups * world * row_blocks(n) * sizeof(uint32_t);
}

extern "C" int dbf_forward_allreduce(const void* A_shard_tiled, const void* B_shard_tiled, const void* a,
                                     const void* mid_shard, const void* b, int scale_dtype, int64_t n,
                                     int64_t k_shard, int64_t m, const void* X, int x_dtype, int64_t batch,
                                     int64_t ldx, void* Y, int y_dtype, int64_t ldy, const uint64_t* peer_recv,
                                     const uint64_t* peer_flags, int world, int rank, uint32_t* epoch_counter,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!A_shard_tiled || !B_shard_tiled || !a || !mid_shard || !b || !X || !Y || !peer_recv || !peer_flags ||
      n < 1 || k_shard < 1 || m < 1 || batch < 1 || ldx < m || ldy < n || world < 1 || rank < 0 ||
      rank >= world || !epoch_counter || !io_dtype_ok(x_dtype) || !io_dtype_ok(y_dtype) ||
      !scale_dtype_ok(scale_dtype) || n > INT32_MAX)
    return DBF_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < dbf_forward_workspace_bytes(n, k_shard, m, batch))
    return DBF_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  float* t = (float*)workspace;
  uint8_t* fw = (uint8_t*)workspace + align256((size_t)batch * k_shard * sizeof(float));
  const size_t fwb = workspace_bytes - align256((size_t)batch * k_shard * sizeof(float));
  // GEMV1 on the local shard: t_g = mid_g * (B_g . (b * x)), no communication
  GemvParams p1 = make_params(B_shard_tiled, k_shard, m, X, x_dtype, ldx, b, mid_shard, scale_dtype,
                              t, DBF_F32, k_shard);
  p1.bump = epoch_counter;  // this call's epoch = counter + 1, visible to GEMV2 by stream order
  int st = run_gemv(p1, (int)batch, s, fw, fwb);
  if (st != DBF_OK) return st;
  // GEMV2 with the all-reduce in its epilogue: partial rows pushed to every rank as they are
  // produced, each row block combined as soon as all ranks have released it
  GemvParams p2 = make_params(A_shard_tiled, n, k_shard, t, DBF_F32, k_shard, nullptr, nullptr,
                              scale_dtype, nullptr, DBF_F32, n);
  p2.ar_world = world;
  p2.ar_rank = rank;
  p2.ar_epoch = epoch_counter;
  p2.ar_bt = (int)batch;
  p2.ar_recv = peer_recv;
  p2.ar_flags = peer_flags;
  p2.ar_a = a;
  p2.ar_y = Y;
  p2.ar_ldy = ldy;
  p2.ar_ydt = y_dtype;
  return run_gemv(p2, (int)batch, s, fw, fwb);
}

namespace dbf {
__global__ void finalize_kernel(const float* __restrict__ P, const void* a, int sdt, int64_t n,
                                int64_t batch, void* Y, int ydt, int64_t ldy) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * batch) return;
  const int64_t bi = i / n, r = i % n;
  store_any(Y, ydt, bi * ldy + r, (double)P[i] * load_any(a, sdt, r));
}
}  // namespace dbf

extern "C" int dbf_finalize_partial(const float* P, const void* a, int scale_dtype, int64_t n,
                                    int64_t batch, void* Y, int y_dtype, int64_t ldy, void* stream) {
  if (!P || !a || !Y || n < 1 || batch < 1 || ldy < n || !io_dtype_ok(y_dtype) ||
      !scale_dtype_ok(scale_dtype))
    return DBF_ERR_INVALID_ARGUMENT;
  finalize_kernel<<<(unsigned)ceil_div(n * batch, 256), 256, 0, (cudaStream_t)stream>>>(
      P, a, scale_dtype, n, batch, Y, y_dtype, ldy);
  return check_launch();
}
