// DBF decode engine: a whole chain of DBF layer forwards in ONE persistent kernel.
//
// Per-layer kernels pay a grid launch + drain per GEMV (4 us back-to-back on B200, ~2 us in a
// graph), which is 3-10x the HBM time of a 7B layer at 2 bits/weight (0.7-1.8 us).  Here one
// CTA per SM runs the whole program (include/dbf_b200.h, dbf_engine_program):
//
//   warp W (producer)    walks this CTA's unit list and streams every unit's packed signs
//                        into a shared-memory ring with cp.async.bulk (TMA bulk copies,
//                        mbarrier complete_tx).  It never waits on activations, so the weights
//                        of the next layers are already in flight while a layer waits for its
//                        input vector -- HBM stays busy across the layer dependencies.
//   warps 0..W-1         (consumers) per unit: quantize the input vector into int8 digit-plane
//                        B fragments (once per segment), then the int8 tensor-core sign GEMV of
//                        decode.cu from the ring, cross-warp integer reduction, epilogue with the
//                        output scale, and publish the 16 outputs as LL words.
//
// Inter-CTA dependencies use an LL ("low latency", as in NCCL's LL protocol) handoff: each
// produced value is written as one 64-bit word {fp32 value, 32-bit epoch}; consumers poll the
// words themselves, so there is no separate flag, fence or counter round trip.  Epochs are
// run_counter * nvectors + vector + 1, advanced by a one-thread kernel after every launch, so
// LL buffers never need clearing.
//
// Arithmetic is identical to decode.cu (same quantization and exact integer sums), so the
// engine's outputs equal a chain of dbf_forward calls bit for bit.
#include <algorithm>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace dbf {
namespace engine {

constexpr int kWarps = 14;                    // consumer warps (+ 1 finalizer + 1 producer = 4 per SMSP)
constexpr int kFinWarp = kWarps;              // finalizer warp index
constexpr int kDeal = 4;                      // chunks per dealt block (round-robin over warps)
constexpr int kCycle = kWarps * kDeal;        // chunks per full dealing cycle
constexpr int kProdWarp = kWarps + 1;         // producer warp index
constexpr int kConsumers = kWarps * 32;
constexpr int kThreads = kConsumers + 64;     // + finalizer warp + producer warp
constexpr int kSlotBytes = 16384;             // one ring slot = 32 chunks of 512 B
constexpr int kSlotChunks = kSlotBytes / kChunkBytes;
constexpr int kRegGroups = 6;                 // register-resident 4-column groups per thread
constexpr int kMaxSmem = 227 * 1024;
constexpr int kMinSlots = 4;
constexpr int kMaxSlots = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}
__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void st_ll(unsigned long long* p, float v, uint32_t epoch) {
  const unsigned long long w = ((unsigned long long)epoch << 32) | (unsigned long long)__float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }
__device__ __forceinline__ void red_add_s32(int* p, int v) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float ld_scale(const void* p, int dt, int i) {
  return dt == DBF_F16 ? __half2float(((const __half*)p)[i]) : ((const float*)p)[i];
}

// Plain (kind 0) vector: the 4 values of group q (columns 4q..4q+3, zero beyond cols).
__device__ __forceinline__ void load_plain(const void* data, int dtype, int cols, int q, float (&u)[4]) {
  const int j0 = 4 * q;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int j = j0 + e;
    u[e] = j < cols ? (dtype == DBF_F16 ? __half2float(((const __half*)data)[j]) : ((const float*)data)[j]) : 0.f;
  }
}
__device__ __forceinline__ void ld_ll4(const unsigned long long* w, unsigned long long (&x)[4]) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x[0]), "=l"(x[1]) : "l"(w));
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x[2]), "=l"(x[3]) : "l"(w + 2));
}
// LL group check: every element below `cols` must carry the expected epoch.
__device__ __forceinline__ bool ll_take(const unsigned long long (&x)[4], int j0, int cols, uint32_t epoch,
                                        float (&u)[4]) {
  bool ok = true;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool in = j0 + e < cols;
    ok &= !in || (uint32_t)(x[e] >> 32) == epoch;
    u[e] = in ? __uint_as_float((uint32_t)x[e]) : 0.f;
  }
  return ok;
}
// Input of a run, resolved into registers once per prepare.
struct InSpec {
  const void* x;
  const void* iscale;
  int kind, dtype, scale_dtype, cols;
};
__device__ __forceinline__ void apply_iscale(const InSpec& in, int q, float (&u)[4]) {
  if (!in.iscale) return;
  const int j0 = 4 * q;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (j0 + e < in.cols) u[e] *= ld_scale(in.iscale, in.scale_dtype, j0 + e);
}
// One group, blocking (used for groups beyond the register-resident ones).
__device__ __forceinline__ void load_group(const InSpec& in, int q, uint32_t epoch, float (&u)[4]) {
  if (in.kind == 1) {
    unsigned long long x[4];
    const unsigned long long* w = (const unsigned long long*)in.x + 4 * q;
    do {
      ld_ll4(w, x);
    } while (!ll_take(x, 4 * q, in.cols, epoch, u));
  } else {
    load_plain(in.x, in.dtype, in.cols, q, u);
  }
  apply_iscale(in, q, u);
}

constexpr int kRedBufs = 16;                  // per-unit partial-sum ring depth (power of 2)

struct Smem {
  uint8_t* ring;
  uint8_t* xfrag;
  long long* red;   // [kRedBufs][kWarps][16]
  int* red_cnt;     // [kRedBufs] arrivals of the unit currently in each buffer
  int* red_fin;     // [kRedBufs] units finalized from each buffer
  long long* run_T; // [2*kRedBufs] T of the run (by run sequence), for the finalizer
  int* run_F;       // [2*kRedBufs] F of the run
  float* red_max;   // [kWarps]
  long long* red_sum;  // [kWarps]
  uint64_t* full;
  uint64_t* empty;
  dbf_engine_run* hdr;  // [kMaxSlots] run record of the run whose first piece is in that slot
};

// Quantize the segment's input vector into B fragments (SINGLE layout: 16 lanes x 8 B per k-block).
// Returns F (every thread) and T = sum_j X_j (valid in all threads after the final barrier).
__device__ void prepare(const InSpec& in, uint32_t epoch, const Smem& sm, int& F_out, long long& T_out,
                        const uint32_t* ready, uint32_t ready_target) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (in.kind == 1 && ready) {
    // one poller per CTA; the data words' epochs are still checked below
    if (tid == 0) {
      uint32_t c;
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ready) : "memory");
        if ((int)(c - ready_target) >= 0) break;
        __nanosleep(64);
      }
    }
    consumer_sync();
  }
  const int nch = (in.cols + kChunkCols - 1) / kChunkCols;
  const int ngroups = nch * (kChunkCols / 4);
  float u[kRegGroups][4];
  if (in.kind == 1) {
    // issue every group's LL loads back to back, then check; re-poll only the pending groups,
    // again in one batched pass, until all carry this run's epoch
    const unsigned long long* base = (const unsigned long long*)in.x;
    unsigned long long x[kRegGroups][4];
#pragma unroll
    for (int g = 0; g < kRegGroups; ++g)
      if (tid + g * kConsumers < ngroups) ld_ll4(base + 4 * (tid + g * kConsumers), x[g]);
    uint32_t pending = 0;
#pragma unroll
    for (int g = 0; g < kRegGroups; ++g) {
      const int q = tid + g * kConsumers;
      if (q < ngroups && !ll_take(x[g], 4 * q, in.cols, epoch, u[g])) pending |= 1u << g;
    }
    while (pending) {
#pragma unroll
      for (int g = 0; g < kRegGroups; ++g)
        if (pending & (1u << g)) ld_ll4(base + 4 * (tid + g * kConsumers), x[g]);
#pragma unroll
      for (int g = 0; g < kRegGroups; ++g)
        if ((pending & (1u << g)) && ll_take(x[g], 4 * (tid + g * kConsumers), in.cols, epoch, u[g]))
          pending &= ~(1u << g);
    }
  } else {
#pragma unroll
    for (int g = 0; g < kRegGroups; ++g) {
      const int q = tid + g * kConsumers;
      if (q < ngroups) load_plain(in.x, in.dtype, in.cols, q, u[g]);
    }
  }
  float mx = 0.f;
#pragma unroll
  for (int g = 0; g < kRegGroups; ++g) {
    const int q = tid + g * kConsumers;
    if (q < ngroups) {
      apply_iscale(in, q, u[g]);
#pragma unroll
      for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fabsf(u[g][e]));
    }
  }
  for (int q = tid + kRegGroups * kConsumers; q < ngroups; q += kConsumers) {
    float t[4];
    load_group(in, q, epoch, t);
#pragma unroll
    for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fabsf(t[e]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) sm.red_max[warp] = mx;
  consumer_sync();
  float m = 0.f;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) m = fmaxf(m, sm.red_max[w]);
  int F = 0;
  if (m > 0.f) {
    int e;
    frexpf(m, &e);
    F = 22 - e;
    F = F > 125 ? 125 : F;
  }
  const float scale = __int_as_float((F + 127) << 23);
  long long tsum = 0;
  auto emit = [&](int q, const float (&uu)[4]) {
    const int kb = q >> 3, r = kb & 7, tig = q & 3, half = (q >> 2) & 1;
    const uint32_t sr = 1u << (7 - r);
    const uint32_t cr = 0x00808080u - 0x4B400000u * sr;
    uint32_t d[4];
    int ts = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t bits = __float_as_uint(fmaf(uu[e], scale, 12582912.0f));
      ts += (int)(bits - 0x4B400000u);
      d[e] = (bits * sr + cr) ^ 0x00808080u;
    }
    tsum += ts;
    const uint32_t t0 = __byte_perm(d[0], d[1], 0x5140), t1 = __byte_perm(d[0], d[1], 0x7362);
    const uint32_t t2 = __byte_perm(d[2], d[3], 0x5140), t3 = __byte_perm(d[2], d[3], 0x7362);
    uint8_t* base = sm.xfrag + kb * 128 + 4 * half + tig * 8;
    *(uint32_t*)(base + 0) = __byte_perm(t0, t2, 0x5410);
    *(uint32_t*)(base + 32) = __byte_perm(t0, t2, 0x7632);
    *(uint32_t*)(base + 64) = __byte_perm(t1, t3, 0x5410);
    *(uint32_t*)(base + 96) = __byte_perm(t1, t3, 0x7632);
  };
#pragma unroll
  for (int g = 0; g < kRegGroups; ++g) {
    const int q = tid + g * kConsumers;
    if (q < ngroups) emit(q, u[g]);
  }
  for (int q = tid + kRegGroups * kConsumers; q < ngroups; q += kConsumers) {
    float t[4];
    load_group(in, q, epoch, t);
    emit(q, t);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
  if (lane == 0) sm.red_sum[warp] = tsum;
  consumer_sync();
  long long T = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) T += sm.red_sum[w];
  F_out = F;
  T_out = T;
}

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(dbf_engine_program prog, int ring_slots,
                                                            int xfrag_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  Smem sm;
  sm.ring = smem;
  sm.hdr = (dbf_engine_run*)(sm.ring + (size_t)ring_slots * kSlotBytes);
  sm.xfrag = (uint8_t*)(sm.hdr + kMaxSlots);
  sm.red = (long long*)(sm.xfrag + xfrag_bytes);
  sm.red_cnt = (int*)(sm.red + kRedBufs * 32);  // red: kRedBufs x 64 int32
  sm.red_fin = sm.red_cnt + kRedBufs;
  sm.run_T = (long long*)(sm.red_fin + kRedBufs);
  sm.run_F = (int*)(sm.run_T + 2 * kRedBufs);
  sm.red_max = (float*)(sm.run_F + 2 * kRedBufs);
  sm.red_sum = (long long*)(sm.red_max + 16);  // 16 floats: keeps the int64 array 8-byte aligned
  sm.full = (uint64_t*)(sm.red_sum + 16);
  sm.empty = sm.full + kMaxSlots;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kRedBufs) {
    sm.red_cnt[threadIdx.x] = 0;
    sm.red_fin[threadIdx.x] = 0;
  }
  for (int i = threadIdx.x; i < kRedBufs * 64; i += kThreads) ((int*)sm.red)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring_slots; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int r0 = prog.cta_offsets[blockIdx.x], r1 = prog.cta_offsets[blockIdx.x + 1];
  const uint32_t run_ctr = *prog.run_counter;
  const uint32_t ebase = run_ctr * (uint32_t)prog.nvectors + 1u;

  if (warp == kProdWarp) {
    // ---------------- producer: stream each run's packed signs (contiguous) into the ring -----
    // The run record is staged into the header of the run's first slot (consumers read it from
    // shared memory); the next record is prefetched while the current run's pieces are issued.
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int slot = 0;
      uint32_t phase = 0;
      const dbf_engine_run* R = prog.runs;
      // prefetch the fields the producer needs one run ahead (the record itself is bulk-copied)
      const void* n_tiled = nullptr;
      int n_cols = 1, n_units = 0;
      if (r0 < r1) { n_tiled = R[r0].tiled; n_cols = R[r0].cols; n_units = R[r0].nunits; }
      for (int i = r0; i < r1; ++i) {
        const uint8_t* src = (const uint8_t*)n_tiled;
        const int cols = n_cols, nunits = n_units;
        if (i + 1 < r1) { n_tiled = R[i + 1].tiled; n_cols = R[i + 1].cols; n_units = R[i + 1].nunits; }
        const int nch = (cols + kChunkCols - 1) / kChunkCols;
        const int total = nunits * nch;
        for (int p = 0; p < total; p += kSlotChunks) {
          const int n = min(kSlotChunks, total - p);
          mbar_wait(&sm.empty[slot], phase ^ 1u);
          if (p == 0) {
            mbar_arrive_expect_tx(&sm.full[slot], n * kChunkBytes + (int)sizeof(dbf_engine_run));
            bulk_g2s(&sm.hdr[slot], R + i, sizeof(dbf_engine_run), &sm.full[slot], pol);
          } else {
            mbar_arrive_expect_tx(&sm.full[slot], n * kChunkBytes);
          }
          bulk_g2s(sm.ring + (size_t)slot * kSlotBytes, src + (size_t)p * kChunkBytes, n * kChunkBytes,
                   &sm.full[slot], pol);
          if (++slot == ring_slots) { slot = 0; phase ^= 1u; }
        }
      }
    }
    return;
  }

  if (warp == kFinWarp) {
    // ---------------- finalizer: completes units in order as their contributions land -------
    // (exact digit recombination, scales, LL publish + ready-counter bump), so the consumer
    // warps never stall on epilogues and stay close together over the ring.
    const dbf_engine_run* R = prog.runs;
    int seq = 0;
    int dealt = 0;  // chunks dealt before the current run, mod kCycle (mirrors the consumers)
    for (int i = r0; i < r1; ++i) {
      const dbf_engine_run& run = R[i];
      const int rows = run.rows, cols = run.cols, rb = run.rb, nunits = run.nunits;
      const void* oscale = run.oscale;
      const int scale_dtype = run.scale_dtype, out_dtype = run.out_dtype;
      void* out_plain = run.out_plain;
      unsigned long long* ll_out = (unsigned long long*)run.ll_out;
      uint32_t* ready_out = run.ready_out;
      const uint32_t out_epoch = ebase + (uint32_t)run.out_vec;
      const int nch = (cols + kChunkCols - 1) / kChunkCols;
      uint32_t osc_next = 0;
      {
        const int row = rb * 16 + (lane & 15);
        if (oscale && row < rows)
          osc_next = scale_dtype == DBF_F16 ? (uint32_t)__ldg((const unsigned short*)oscale + row)
                                            : __ldg((const uint32_t*)oscale + row);
      }
      const int rs = (i - r0) & (2 * kRedBufs - 1);
      bool have_FT = false;
      int F = 0;
      long long T = 0;
      double inv_scale = 1.0;
      for (int uu = 0; uu < nunits; ++uu, ++seq) {
        const uint32_t osc_raw = osc_next;
        if (uu + 1 < nunits) {  // prefetch the next unit's output scale
          const int row = (rb + uu + 1) * 16 + (lane & 15);
          if (oscale && row < rows)
            osc_next = scale_dtype == DBF_F16 ? (uint32_t)__ldg((const unsigned short*)oscale + row)
                                              : __ldg((const uint32_t*)oscale + row);
        }
        const int rbuf = seq & (kRedBufs - 1);
        // contributors = dealt blocks intersecting the unit (one flush per warp per unit)
        const int v0 = dealt + uu * nch, v1 = v0 + nch - 1;
        int need = v1 / kDeal - v0 / kDeal + 1;
        need = need < kWarps ? need : kWarps;
        while (*(volatile int*)&sm.red_cnt[rbuf] < need) {
        }
        fence_cta();
        if (!have_FT) {  // written by the consumers before their first contribution to this run
          F = *(volatile int*)&sm.run_F[rs];
          T = *(volatile long long*)&sm.run_T[rs];
          inv_scale = __longlong_as_double((long long)(1023 - F) << 52);  // 2^-F
          have_FT = true;
        }
        int* red = (int*)sm.red + rbuf * 64;
        const int row = (rb + uu) * 16 + lane;
        if (lane < 16) {
          int4* pp = (int4*)&red[lane * 4];
          const int4 sum = *pp;
          *pp = make_int4(0, 0, 0, 0);
          if (row < rows) {
            const long long s128 = (long long)sum.x + ((long long)sum.y << 8) + ((long long)sum.z << 16) +
                                   ((long long)sum.w << 24);
            const long long P = 2 * (s128 >> 7) - T;
            const float oscf = oscale ? (scale_dtype == DBF_F16 ? __half2float(__ushort_as_half((unsigned short)osc_raw))
                                                                : __uint_as_float(osc_raw))
                                      : 1.f;
            float fv = (float)((double)P * inv_scale * (double)oscf);
            if (out_dtype == DBF_F16) {
              const __half h = __float2half_rn(fv);
              fv = __half2float(h);
              if (out_plain) ((__half*)out_plain)[row] = h;
            } else if (out_plain) {
              ((float*)out_plain)[row] = fv;
            }
            if (ll_out) st_ll(ll_out + row, fv, out_epoch);
          }
        }
        __syncwarp();
        if (lane == 0) {
          if (ready_out) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ready_out) : "memory");
          sm.red_cnt[rbuf] = 0;
          fence_cta();
          *(volatile int*)&sm.red_fin[rbuf] = seq / kRedBufs + 1;
        }
        __syncwarp();
      }
      dealt = (dealt + nunits * nch) % kCycle;
    }
    return;
  }

  // ---------------- consumers ---------------------------------------------------------------
  // A run's chunks are dealt round-robin over the 15 consumer warps (continuing across runs),
  // so no warp waits for another per unit.  When a warp leaves a unit it drops its partial
  // (int32 shared-memory reductions, exact) into a ring of kRedBufs per-unit accumulators and
  // bumps the unit's arrival count; the finalizer warp completes units in order.
  const int g = lane >> 2, tig = lane & 3;
  const uint2* xlane = (const uint2*)sm.xfrag + (lane & 15);  // lanes 16-31 mirror 0-15 (ignored cols)
  int slot = 0;
  uint32_t phase = 0;
  int cur_seg = -1;
  int F = 0;
  long long T = 0;
  int dealt = 0;      // chunks dealt on this CTA so far, mod kCycle
  int unit_seq = 0;   // units completed on this CTA before the current run
  for (int i = r0; i < r1; ++i) {
    int64_t* tr = prog.trace ? prog.trace + 4 * (size_t)i : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();
    mbar_wait(&sm.full[slot], phase);  // first piece of the run: its header holds the record
    const dbf_engine_run& H = sm.hdr[slot];
    const int rows = H.rows, cols = H.cols, rb = H.rb, nunits = H.nunits;
    if (H.seg != cur_seg) {
      InSpec in;
      in.x = H.x;
      in.iscale = H.iscale;
      in.kind = H.in_kind;
      in.dtype = H.in_dtype;
      in.scale_dtype = H.scale_dtype;
      in.cols = cols;
      prepare(in, ebase + (uint32_t)H.in_vec, sm, F, T, H.ready_in, (run_ctr + 1u) * H.in_producers);
      cur_seg = H.seg;
    }
    if (threadIdx.x == 0) {  // F/T of this run for the finalizer; depth 2*kRedBufs runs is safe:
      // reaching run i+2R means unit seq(i)+2R-1 was flushed, which waited for seq(i)+R-1 done
      sm.run_F[(i - r0) & (2 * kRedBufs - 1)] = F;
      sm.run_T[(i - r0) & (2 * kRedBufs - 1)] = T;
    }
    if (tr && threadIdx.x == 0) tr[1] = gtimer();
    const int nch = (cols + kChunkCols - 1) / kChunkCols;
    const int total = nunits * nch;
    // virtual chunk index v = run chunk + dealt; this warp owns v with (v / kDeal) % kWarps == warp
    int v = warp * kDeal;  // this warp's first block of the cycle
    if (v + kDeal <= dealt) v += kCycle;  // already passed: take the next cycle's block
    else if (v < dealt) v = dealt;        // the run starts inside this warp's block
    int gch = v - dealt;
    int u = gch / nch, cu = gch - u * nch;
    int cur_u = -1;
    int acc[4][4] = {};

    auto flush = [&](int uu) {
      // add this warp's int32 plane sums into the unit's 16x4 accumulator (exact, order-free)
      const int c0 = acc[0][0] + acc[1][0] + acc[2][0] + acc[3][0];
      const int c1 = acc[0][1] + acc[1][1] + acc[2][1] + acc[3][1];
      const int c2 = acc[0][2] + acc[1][2] + acc[2][2] + acc[3][2];
      const int c3 = acc[0][3] + acc[1][3] + acc[2][3] + acc[3][3];
      const int seq = unit_seq + uu;
      const int rbuf = seq & (kRedBufs - 1);
      int* red = (int*)sm.red + rbuf * 64;  // [row 16][plane 4] int32
      while (*(volatile int*)&sm.red_fin[rbuf] != seq / kRedBufs) {
      }
      if (tig < 2) {
        red_add_s32(&red[g * 4 + 2 * tig], c0);
        red_add_s32(&red[g * 4 + 2 * tig + 1], c1);
        red_add_s32(&red[(g + 8) * 4 + 2 * tig], c2);
        red_add_s32(&red[(g + 8) * 4 + 2 * tig + 1], c3);
      }
      __syncwarp();
      fence_cta();
      if (lane == 0) atomicAdd(&sm.red_cnt[rbuf], 1);
    };

    bool first_piece = true;
    for (int pb = 0; pb < total; pb += kSlotChunks) {
      const int pe = min(pb + kSlotChunks, total);
      if (!first_piece) mbar_wait(&sm.full[slot], phase);
      if (tr && threadIdx.x == 0 && first_piece) tr[2] = gtimer();
      first_piece = false;
      const uint4* piece = (const uint4*)(sm.ring + (size_t)slot * kSlotBytes) + lane;
      for (; gch < pe;) {
        if (u != cur_u) {
          if (cur_u >= 0) flush(cur_u);
          cur_u = u;
#pragma unroll
          for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = acc[a][2] = acc[a][3] = 0;
        }
        const uint4 w = piece[(gch - pb) * 32];
        const uint2* xk = xlane + cu * 8 * 16;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint32_t m = 0x01010101u << r;
          const uint2 b = xk[r * 16];
          imma(acc[r & 3], w.x & m, w.y & m, w.z & m, w.w & m, b.x, b.y);
        }
        // next owned chunk: +1 inside the block, else jump to this warp's next block
        int step = 1;
        if (((gch + dealt + 1) % kDeal) == 0) step = 1 + (kWarps - 1) * kDeal;
        gch += step;
        cu += step;
        while (cu >= nch) { cu -= nch; ++u; }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[slot]);
      if (++slot == ring_slots) { slot = 0; phase ^= 1u; }
    }
    if (cur_u >= 0) flush(cur_u);
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
    dealt = (dealt + total) % kCycle;
    unit_seq += nunits;
  }
}

__global__ void advance_run_kernel(uint32_t* run_counter) { *run_counter += 1u; }

int ring_slots_for(int xfrag_bytes) {
  const int fixed = xfrag_bytes + kMaxSlots * (int)sizeof(dbf_engine_run) + kRedBufs * 64 * 4 +
                    2 * kRedBufs * 4 + 2 * kRedBufs * 12 + 16 * 4 + 16 * 8 + 2 * kMaxSlots * 8 + 256;
  int slots = (kMaxSmem - fixed) / kSlotBytes;
  return std::min(slots, kMaxSlots);
}
int xfrag_bytes_for(int max_cols) {
  const int nch = (max_cols + kChunkCols - 1) / kChunkCols;
  return nch * 8 * 128;
}
size_t smem_bytes(int slots, int xfrag_bytes) {
  return (size_t)slots * kSlotBytes + kMaxSlots * sizeof(dbf_engine_run) + xfrag_bytes +
         kRedBufs * 64 * 4 + 2 * kRedBufs * 4 + 2 * kRedBufs * 12 + 16 * 4 + 16 * 8 + 2 * kMaxSlots * 8 + 64;
}

}  // namespace engine
}  // namespace dbf

using namespace dbf;

static_assert(sizeof(dbf_engine_run) == 128, "run record must be 128 bytes");

extern "C" int dbf_engine_build_runs(const dbf_engine_segment* segments, int32_t nsegments,
                                     const dbf_engine_vector* vectors, int32_t nvectors, const int32_t* runs,
                                     int32_t nruns, uint32_t* ready, dbf_engine_run* out) {
  if (!segments || !vectors || !runs || !out || nsegments < 1 || nvectors < 1 || nruns < 0)
    return DBF_ERR_INVALID_ARGUMENT;
  // units producing each vector (one segment writes each LL vector)
  std::vector<uint32_t> producers(nvectors, 0);
  for (int s = 0; s < nsegments; ++s) {
    const dbf_engine_segment& g = segments[s];
    if (g.rows < 1 || g.cols < 1 || !g.tiled || g.in_vec < 0 || g.in_vec >= nvectors || g.out_vec >= nvectors)
      return DBF_ERR_INVALID_ARGUMENT;
    if (g.out_vec >= 0) {
      if (vectors[g.out_vec].kind != 1) return DBF_ERR_INVALID_ARGUMENT;
      producers[g.out_vec] += (uint32_t)((g.rows + kRowBlock - 1) / kRowBlock);
    }
  }
  for (int i = 0; i < nruns; ++i) {
    const int seg = runs[3 * i], rb = runs[3 * i + 1], n = runs[3 * i + 2];
    if (seg < 0 || seg >= nsegments || rb < 0 || n < 1) return DBF_ERR_INVALID_ARGUMENT;
    const dbf_engine_segment& g = segments[seg];
    if ((int64_t)(rb + n) * kRowBlock > (int64_t)((g.rows + kRowBlock - 1) / kRowBlock) * kRowBlock)
      return DBF_ERR_SHAPE;
    const dbf_engine_vector& vin = vectors[g.in_vec];
    if (vin.len != g.cols) return DBF_ERR_SHAPE;
    dbf_engine_run r;
    memset(&r, 0, sizeof(r));
    const int64_t nch = chunks(g.cols);
    r.tiled = (const uint8_t*)g.tiled + (size_t)rb * nch * kChunkBytes;
    r.x = vin.data;
    r.iscale = g.iscale;
    r.oscale = g.oscale;
    r.out_plain = g.out_plain;
    r.ll_out = g.out_vec >= 0 ? vectors[g.out_vec].data : nullptr;
    r.ready_in = (vin.kind == 1 && ready) ? ready + g.in_vec : nullptr;
    r.ready_out = (g.out_vec >= 0 && ready) ? ready + g.out_vec : nullptr;
    r.rows = g.rows;
    r.cols = g.cols;
    r.rb = rb;
    r.nunits = n;
    r.seg = seg;
    r.in_kind = vin.kind;
    r.in_dtype = vin.dtype;
    r.scale_dtype = g.scale_dtype;
    r.out_dtype = g.out_dtype;
    r.in_vec = g.in_vec;
    r.out_vec = g.out_vec;
    r.in_producers = producers[g.in_vec];
    out[i] = r;
  }
  return DBF_OK;
}

extern "C" int dbf_engine_smem_bytes(int32_t max_cols, size_t* bytes) {
  if (max_cols < 1 || !bytes) return DBF_ERR_INVALID_ARGUMENT;
  const int xb = engine::xfrag_bytes_for(max_cols);
  const int slots = engine::ring_slots_for(xb);
  if (slots < engine::kMinSlots) return DBF_ERR_UNSUPPORTED;
  *bytes = engine::smem_bytes(slots, xb);
  return DBF_OK;
}

extern "C" int dbf_engine_occupancy(int32_t max_cols, int32_t* blocks_per_sm, int32_t* regs_per_thread) {
  if (!blocks_per_sm || !regs_per_thread || max_cols < 1) return DBF_ERR_INVALID_ARGUMENT;
  const int xb = engine::xfrag_bytes_for(max_cols);
  const int slots = engine::ring_slots_for(xb);
  if (slots < engine::kMinSlots) return DBF_ERR_UNSUPPORTED;
  cudaError_t e = cudaFuncSetAttribute(engine::engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       engine::kMaxSmem);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, engine::engine_kernel);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  *regs_per_thread = fa.numRegs;
  int nb = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, engine::engine_kernel, engine::kThreads,
                                                    engine::smem_bytes(slots, xb));
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  *blocks_per_sm = nb;
  return DBF_OK;
}

extern "C" int dbf_engine_launch(const dbf_engine_program* program, void* stream) {
  if (!program || !program->runs || !program->cta_offsets || !program->run_counter || program->grid < 1 ||
      program->max_cols < 1)
    return DBF_ERR_INVALID_ARGUMENT;
  const int xb = engine::xfrag_bytes_for(program->max_cols);
  const int slots = engine::ring_slots_for(xb);
  if (slots < engine::kMinSlots) return DBF_ERR_UNSUPPORTED;
  const size_t smem = engine::smem_bytes(slots, xb);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(engine::engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         engine::kMaxSmem);
    if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
    configured = true;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(program->grid);
  cfg.blockDim = dim3(engine::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  dbf_engine_program prog = *program;
  cudaError_t e = cudaLaunchKernelEx(&cfg, engine::engine_kernel, prog, slots, xb);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  engine::advance_run_kernel<<<1, 1, 0, s>>>(program->run_counter);
  return check_launch();
}
