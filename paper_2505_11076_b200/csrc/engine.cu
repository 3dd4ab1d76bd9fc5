// DBF decode engine: a whole chain of DBF layer forwards in ONE persistent kernel.
//
// Per-layer kernels pay a grid launch + drain per GEMV (4 us back-to-back on B200, ~2 us in a
// graph), which is 3-10x the HBM time of a 7B layer at 2 bits/weight (0.7-1.8 us).  Here one
// CTA per SM runs the whole program (include/dbf_b200.h, dbf_engine_program) -- a list of RUNS
// (consecutive 16-row units of one segment) per CTA, in stage order:
//
//   producer warp        streams every run's packed signs (+ its 128-byte record) into a
//                        shared-memory ring with cp.async.bulk (mbarrier complete_tx).  It never
//                        waits on activations, so the next layers' weights are in flight while a
//                        layer waits for its input.
//   16 compute warps     warp w OWNS the 256-column chunks c = w, w+16, ... of the run's input.
//                        Per chunk it polls the chunk's LL words straight from L2 (streaming: a
//                        chunk is processed as soon as ITS producers are done), quantizes the 256
//                        values to a 13-bit grid relative to the CHUNK's max |value| (|X| <= 4079;
//                        warp-local: no CTA-wide barrier, no global max), builds the two int8
//                        digit-plane B fragments, and runs the int8 tensor-core sign GEMV of every unit of the
//                        run against that chunk.  The chunk's exact integer sum is scaled by
//                        2^-F_c and accumulated in fp32 registers, per unit, in chunk order.
//   finalizer warps      warp 15 - u sums the 16 warps' partials of unit u in warp order
//                        (deterministic), applies the output scale and publishes fp16 outputs as
//                        LL words (plain stores for outputs no later stage reads).
//
// Inter-CTA dependencies use an LL ("low latency", as in NCCL's LL protocol) handoff: each value
// is one 32-bit word {fp16 value, 16-bit epoch}; consumers poll the words themselves, so there is
// no separate flag, fence or counter round trip.  Epochs are (launch * nvectors + vector) mod
// 65535 + 1; the last CTA of a launch advances the launch counter, so LL buffers never need
// clearing (a stale word always carries the previous launch's epoch).
#include <algorithm>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace dbf {
namespace engine {

constexpr int kWarps = 16;                    // compute warps
constexpr int kProdWarp = kWarps;             // producer warp index (first warp of the last warpgroup)
// 16 compute warps + one producer WARPGROUP (warp 16 streams, 17-19 only hand their registers
// back): the producer warpgroup drops to kProdRegs with setmaxnreg and the compute warpgroups
// grow to kComputeRegs, where 17 warps at launch cap every thread at 96 (5 warps on one SM
// sub-partition).  120 would fit the register file on paper but setmaxnreg.inc never returns
// with it on B200 (measured); 112 does.
constexpr int kThreads = (kWarps + 4) * 32;
#ifndef DBF_COMPUTE_REGS
#define DBF_COMPUTE_REGS 112  // setmaxnreg for the 16 compute warps (the producer warpgroup drops to 24)
#endif
constexpr int kProdRegs = 24, kComputeRegs = DBF_COMPUTE_REGS;
// setmaxnreg.inc only draws on registers the producer warpgroup released (launch allocation 96 per
// thread at 640 threads): asking for more blocks the compute warps forever (120 measured: hang)
static_assert(16 * (kComputeRegs - 96) <= 4 * (96 - kProdRegs), "compute warps would wait for registers forever");
constexpr int kSlotBytes = 16384;             // one ring slot = 32 chunks of 512 B
#ifndef DBF_CHAINS
#define DBF_CHAINS 1  // accumulator chains per unit (1, 2, 4 measured within 1 %; 1 issues fewest)
#endif
constexpr int kMaxUnits = 8;                  // units per run (the host splits longer runs)
// 4-token runs keep at most 4 units: their accumulators, token pairs and quantizer state would not
// fit the 112 registers otherwise (spills on the run-start path), and the smaller partial buffer
// leaves room for two quantized chunks per warp (inputs up to 32 chunks quantized once per CTA)
#ifndef DBF_NB4_UNITS
#define DBF_NB4_UNITS 4
#endif
template <int NB> constexpr int max_units() { return NB == 4 ? DBF_NB4_UNITS : kMaxUnits; }
inline int max_units_of(int nb) { return nb == 4 ? DBF_NB4_UNITS : kMaxUnits; }
#ifndef DBF_POLL_NS
#define DBF_POLL_NS 32
#endif
constexpr int kPollSleepNs = DBF_POLL_NS;     // back-off between LL polls of a not-yet-published chunk
#ifndef DBF_PACE_NS
#define DBF_PACE_NS 1200
#endif
#ifndef DBF_PACE_AHEAD
#define DBF_PACE_AHEAD 1
#endif
constexpr int kPaceNs = DBF_PACE_NS, kPaceAhead = DBF_PACE_AHEAD;  // producer pacing (stream_runs)
constexpr int kMaxSmem = 227 * 1024;
constexpr int kMinSlots = 4;
constexpr int kMaxSlots = 16;
// Per token of a batch (NB tokens share every MMA: B column n = 2*token + digit plane):
constexpr float kQScale = 4079.f / 4096.f;    // keeps 8 * |X| below the two-digit limit 32640
constexpr float kQInv = 4096.f / 4079.f;
// chunk exponent of a chunk holding inf / NaN: 1 / (2^F kQScale) = 2^(127 - F) overflows to inf
constexpr int kBadF = -128;
// status bits of a launch (run_counter[2], sticky until the host clears them)
constexpr uint32_t kStatusNonFinite = 1u;  // an input chunk held inf / NaN (its outputs are NaN)
constexpr uint32_t kStatusOverflow = 2u;   // a value rounded to fp16 overflowed (|v| > 65504)
constexpr int kChunkQBytes1 = 8 * 64;         // one quantized chunk: 8 k-blocks x (2 planes x 4 lanes x 8 B)
constexpr int kQScrFT = 32;                   // scratch bytes per chunk for F, T of up to 4 tokens
inline int part_floats(int nb) { return kWarps * max_units_of(nb) * 16 * nb; }  // one partial buffer
// chunks a warp keeps quantized for reuse by the next run on the same input (a stage split over
// several runs of one CTA): inputs up to 16 * xs_chunks chunks
#ifndef DBF_XS_CHUNKS1
#define DBF_XS_CHUNKS1 4  // 64 chunks: the 70B gate/up A stage (50 chunks, 3 runs per CTA) quantizes once
#endif
#ifndef DBF_XS_CHUNKS1_MAX
#define DBF_XS_CHUNKS1_MAX 7  // 112 chunks: the 70B down.B stage (m = 28672) quantizes its input once
#endif
// batch 1 sizes the quantized-chunk store from the program's widest input (one slot per 16
// chunks, so a stage of any width up to 16 * DBF_XS_CHUNKS1_MAX chunks quantizes once per CTA);
// the ring gets the rest of shared memory
inline int xs_chunks_of(int nb, int max_cols = 0) {
  // 2 tokens: 64 chunks; 4 tokens: 32 chunks when the widest unit leaves a deep enough ring
  // (<= 16384 columns: 7B, 13B), else 16 (the 70B's 57 KB units want the 10-slot ring)
  if (nb == 2) return 4;
  if (nb == 4) return chunks(max_cols) <= 64 ? 2 : 1;
  const int need = (int)((chunks(max_cols) + kWarps - 1) / kWarps);
  return need <= DBF_XS_CHUNKS1 ? DBF_XS_CHUNKS1 : DBF_XS_CHUNKS1_MAX;  // the two batch-1 instantiations
}

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
__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm(  // no side effects: let the compiler interleave independent MMA chains
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void st_ll16(uint32_t* p, __half v, uint32_t epoch) {
  const uint32_t w = (epoch << 16) | (uint32_t)__half_as_ushort(v);
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 ld_ll16x4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
#ifdef DBF_LL_TRACE
__device__ unsigned long long g_ll_rtt[2];  // debug build: sum of LL poll round trips (ns), count
#endif
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// non-blocking loads of raw scale bits (the consumer converts them when it needs the value)
__device__ __forceinline__ uint32_t ld_nc_u16(const unsigned short* p) {
  unsigned short v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_scale(const void* p, int dt, int i) {
  return dt == DBF_F16 ? __half2float(((const __half*)p)[i]) : ((const float*)p)[i];
}
// epoch of vector `vec` in this launch: (launch * nvectors + vec) mod 65535 + 1, from the launch's
// base (launch * nvectors) mod 65535
__device__ __forceinline__ uint32_t epoch16(uint32_t base, int vec) {
  return (base + (uint32_t)vec) % 65535u + 1u;
}

struct Smem {
  uint8_t* ring;
  dbf_engine_run* hdr;  // [kMaxSlots] record of the run whose first piece is in that slot
  uint8_t* xs;          // [kWarps][kXsBytes]
  float* part;          // [2][kWarps][max_units][NB][16]
  uint64_t* full;
  uint64_t* empty;
};

// A run's input vector, resolved into registers once per run.
struct InSpec {
  const void* x;
  const void* iscale;
  int kind, dtype, sdt, cols;
  int64_t tstride;  // elements between consecutive tokens of the vector
};
__device__ __forceinline__ InSpec token_of(const InSpec& in, int t) {
  InSpec o = in;
  const int esz = in.kind == 1 ? 4 : (in.dtype == DBF_F16 ? 2 : 4);
  o.x = (const char*)in.x + (int64_t)t * in.tstride * esz;
  return o;
}

// The 4 input scales of columns col0..col0+3 (1 when there is no input scale, 0 beyond cols).
__device__ __forceinline__ void load_scale4(const InSpec& in, int col0, float (&s)[4]) {
  if (!in.iscale) {
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = 1.f;
    return;
  }
  if (col0 + 3 < in.cols) {
    if (in.sdt == DBF_F16) {
      const uint2 v = __ldg((const uint2*)((const __half*)in.iscale + col0));
      const float2 a = __half22float2(*(const __half2*)&v.x), b = __half22float2(*(const __half2*)&v.y);
      s[0] = a.x, s[1] = a.y, s[2] = b.x, s[3] = b.y;
    } else {
      const float4 v = __ldg((const float4*)((const float*)in.iscale + col0));
      s[0] = v.x, s[1] = v.y, s[2] = v.z, s[3] = v.w;
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] = col0 + e < in.cols ? ld_scale(in.iscale, in.sdt, col0 + e) : 0.f;
}

// Decode 4 LL words {fp16, epoch16} of columns col0..col0+3 (0 beyond cols); true if all carry epoch.
__device__ __forceinline__ bool ll_group(const uint4 v, int col0, int cols, uint32_t epoch, float (&u)[4]) {
  const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
  bool ok = true;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool inb = col0 + e < cols;
    ok &= !inb || (vv[e] >> 16) == epoch;
    u[e] = inb ? __half2float(__ushort_as_half((unsigned short)(vv[e] & 0xFFFFu))) : 0.f;
  }
  return ok;
}

// Load the 4 values of columns col0..col0+3; for LL vectors also report whether all carry `epoch`.
// Columns >= cols read as 0.
__device__ __forceinline__ bool load_group(const InSpec& in, int col0, uint32_t epoch, float (&u)[4]) {
  if (in.kind == 1) {
    const uint4 v = ld_ll16x4((const uint32_t*)in.x + col0);  // LL vectors are padded to whole chunks
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
    bool ok = true;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool inb = col0 + e < in.cols;
      ok &= !inb || (vv[e] >> 16) == epoch;
      u[e] = inb ? __half2float(__ushort_as_half((unsigned short)(vv[e] & 0xFFFFu))) : 0.f;
    }
    return ok;
  }
  if (col0 + 3 < in.cols && in.dtype == DBF_F16 && (((uintptr_t)in.x & 7) == 0)) {
    const uint2 v = __ldg((const uint2*)((const __half*)in.x + col0));
    const float2 a = __half22float2(*(const __half2*)&v.x), b = __half22float2(*(const __half2*)&v.y);
    u[0] = a.x, u[1] = a.y, u[2] = b.x, u[3] = b.y;
    return true;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int j = col0 + e;
    u[e] = j < in.cols ? (in.dtype == DBF_F16 ? __half2float(((const __half*)in.x)[j]) : ((const float*)in.x)[j])
                       : 0.f;
  }
  return true;
}

// Scale and quantize one chunk (this lane: groups lane and lane + 32) into the warp's
// B-fragment scratch; see quantize_chunk.  Returns F and T = sum_j X_j.
__device__ __forceinline__ void emit_digits(float (&u)[2][4], const float (&sc)[2][4], uint8_t* xs, int kb_stride,
                                            int lane, int& F_out, int& T_out) {
  // max |u| with NaN propagation (max.NaN: a NaN anywhere makes the max NaN; fmaxf would drop it)
  float mx = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      u[h][e] *= sc[h][e];
      mx = fmax_nan(mx, fabsf(u[h][e]));
    }
  }
  // |u| >= 0 (or NaN): the float bits order like unsigned integers, inf / NaN >= 0x7F800000
  const uint32_t mxb = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
  int F = 0;
  float scale;
  if (mxb >= 0x7F800000u) {
    // a non-finite input (or an fp16 overflow upstream): the chunk's digits are zero and
    // F = kBadF makes 1 / (2^F kQScale) = inf, so every output this chunk feeds is NaN instead of
    // a finite value computed from garbage digits; the launch's status word records it
    F = kBadF;
    scale = 0.f;
  } else {
    if (mxb != 0u) {
      // mx in [2^(e-1), 2^e) with e = biased exponent - 126 (mx is a normal float: fp16 inputs
      // times fp16/fp32 scales stay far above 2^-126)  ->  |X| <= 4096 * kQScale <= 4079
      const int e = (int)(mxb >> 23) - 126;
      F = 12 - e;
      F = F > 125 ? 125 : (F < -125 ? -125 : F);
    }
    scale = __int_as_float((F + 127) << 23) * kQScale;
  }
  int ts = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h;
    const int kb = q >> 3, tig = q & 3, half = (q >> 2) & 1;
    const int sh = 3 - (kb & 3);  // Y = X * 2^(3-t), |Y| <= 32632 < 32640 (two balanced digits)
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // round to nearest even through the fp32 adder (|X| <= 4079 << 2^22): no F2I on the
      // quarter-rate conversion pipe
      const int X = __float_as_int(fmaf(u[h][e], scale, 12582912.f)) - 0x4B400000;
      ts += X;
      v[e] = (uint32_t)((X << sh) + 0x8080);  // bytes 0,1 = balanced digits + 128
    }
    const uint32_t lo = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);
    uint8_t* base = xs + kb * kb_stride + 4 * half + tig * 8;
    *(uint32_t*)(base + 0) = lo ^ 0x80808080u;   // plane 0 -> MMA column 0 (lanes 0-3)
    *(uint32_t*)(base + 32) = hi ^ 0x80808080u;  // plane 1 -> MMA column 1 (lanes 4-7)
  }
  ts = __reduce_add_sync(0xffffffffu, ts);
  __syncwarp();  // the digit stores above are visible to every lane of the warp
  F_out = F;
  T_out = ts;
}

// Quantize chunk c of the run's input (256 columns, warp-local) into this warp's B-fragment
// scratch.  X_j = round(x_j * 2^F * kQScale) on a 13-bit grid relative to the CHUNK max
// (|X| <= 4079); the MMA A bytes are 2^t * bit_j for k-block r = 4s + t (the packed word
// pre-shifted by 4s: one shift per word serves four k-blocks), so the B operand carries
// Y_j = X_j * 2^(3-t) as two balanced int8 digits (planes = MMA columns 0, 1; |Y| < 32640 keeps
// both digits in [-128, 127]) and every k-block contributes 8 * sum bit_j X_j alike.
// Returns F and T = sum_j X_j.
__device__ __forceinline__ void quantize_chunk(const InSpec& in, int c, uint32_t epoch, uint8_t* xs, int kb_stride,
                                               int& F_out, int& T_out, int64_t* dbg = nullptr) {
  const int lane = threadIdx.x & 31;
  float u[2][4], sc[2][4];
  const int c0 = c * kChunkCols;
  // groups q = lane and lane + 32 (64 groups of 4 columns per chunk).  fp16 scales of whole
  // groups are loaded as raw bits before the poll and converted after it (converting here would
  // hold the first poll back by a full round trip); other scale layouts load directly.
  const bool raw_sc = in.iscale && in.sdt == DBF_F16 && c0 + 4 * (lane + 32) + 3 < in.cols;
  uint2 sr0 = make_uint2(0, 0), sr1 = make_uint2(0, 0);
  if (raw_sc) {
    sr0 = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * lane));
    sr1 = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * (lane + 32)));
  } else {
    load_scale4(in, c0 + 4 * lane, sc[0]);
    load_scale4(in, c0 + 4 * (lane + 32), sc[1]);
  }
  int npoll = 0;
  if (dbg && lane == 0) dbg[0] = gtimer();
  for (;;) {
    const bool ok0 = load_group(in, c0 + 4 * lane, epoch, u[0]);
    const bool ok1 = load_group(in, c0 + 4 * (lane + 32), epoch, u[1]);
    ++npoll;
    if (__all_sync(0xffffffffu, ok0 && ok1)) break;
    if (kPollSleepNs) __nanosleep(kPollSleepNs);
  }
  if (dbg && lane == 0) { dbg[1] = gtimer(); dbg[2] = npoll; }
  if (raw_sc) {
    const float2 a0 = __half22float2(*(const __half2*)&sr0.x), b0 = __half22float2(*(const __half2*)&sr0.y);
    const float2 a1 = __half22float2(*(const __half2*)&sr1.x), b1 = __half22float2(*(const __half2*)&sr1.y);
    sc[0][0] = a0.x, sc[0][1] = a0.y, sc[0][2] = b0.x, sc[0][3] = b0.y;
    sc[1][0] = a1.x, sc[1][1] = a1.y, sc[1][2] = b1.x, sc[1][3] = b1.y;
  }
  emit_digits(u, sc, xs, kb_stride, lane, F_out, T_out);
}

// Batch 1, LL input: the next chunk's LL words (and raw fp16 scales) are loaded while the
// current chunk's MMAs run, so a warp that owns several chunks of a run pays the L2 round trip
// once (the words are re-polled only if they were not yet published when prefetched).
struct ChunkFetch {
  uint4 v[2];
  uint2 s[2];
};
__device__ __forceinline__ void fetch_issue(const InSpec& in, int c, int lane, ChunkFetch& f) {
  const int c0 = c * kChunkCols;
  f.v[0] = ld_ll16x4((const uint32_t*)in.x + c0 + 4 * lane);
  f.v[1] = ld_ll16x4((const uint32_t*)in.x + c0 + 4 * (lane + 32));
  if (in.iscale && in.sdt == DBF_F16 && c0 + 4 * (lane + 32) + 3 < in.cols) {
    f.s[0] = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * lane));
    f.s[1] = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * (lane + 32)));
  }
}
__device__ __forceinline__ void quantize_fetched(const InSpec& in, int c, uint32_t epoch, uint8_t* xs, int& F_out,
                                                 int& T_out, const ChunkFetch& f) {
  const int lane = threadIdx.x & 31;
  float u[2][4], sc[2][4];
  const int c0 = c * kChunkCols;
  const bool ok0 = ll_group(f.v[0], c0 + 4 * lane, in.cols, epoch, u[0]);
  const bool ok1 = ll_group(f.v[1], c0 + 4 * (lane + 32), in.cols, epoch, u[1]);
  if (!__all_sync(0xffffffffu, ok0 && ok1)) {
      for (;;) {  // not all published when prefetched: poll as usual
#ifdef DBF_LL_TRACE
      const long long t0 = gtimer();
#endif
      const bool p0 = load_group(in, c0 + 4 * lane, epoch, u[0]);
      const bool p1 = load_group(in, c0 + 4 * (lane + 32), epoch, u[1]);
      const bool done = __all_sync(0xffffffffu, p0 && p1);
#ifdef DBF_LL_TRACE
      if (lane == 0) { atomicAdd(&g_ll_rtt[0], (unsigned long long)(gtimer() - t0)); atomicAdd(&g_ll_rtt[1], 1ull); }
#endif
      if (done) break;
      if (kPollSleepNs) __nanosleep(kPollSleepNs);
    }
  }
  if (in.iscale && in.sdt == DBF_F16 && c0 + 4 * (lane + 32) + 3 < in.cols) {
    const float2 a0 = __half22float2(*(const __half2*)&f.s[0].x), b0 = __half22float2(*(const __half2*)&f.s[0].y);
    const float2 a1 = __half22float2(*(const __half2*)&f.s[1].x), b1 = __half22float2(*(const __half2*)&f.s[1].y);
    sc[0][0] = a0.x, sc[0][1] = a0.y, sc[0][2] = b0.x, sc[0][3] = b0.y;
    sc[1][0] = a1.x, sc[1][1] = a1.y, sc[1][2] = b1.x, sc[1][3] = b1.y;
  } else {
    load_scale4(in, c0 + 4 * lane, sc[0]);
    load_scale4(in, c0 + 4 * (lane + 32), sc[1]);
  }
  emit_digits(u, sc, xs, 64, lane, F_out, T_out);
}

// NB > 1 tokens: the same for every present token of chunk c, polling two tokens at a time
// (their loads are in flight together instead of one round trip per token); absent tokens get
// zero digits.
template <int NB>
__device__ __forceinline__ void emit_tokens(float (&u)[2][2][4], const float (&sc)[2][4], uint8_t* xq, int t0,
                                            int batch, int lane, int (&F)[NB], int (&T)[NB]) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = t0 + i;
    if (t < batch) {
      emit_digits(u[i], sc, xq + t * 64, NB * 64, lane, F[t], T[t]);
    } else {  // absent token: zero digits
      for (int e = lane; e < 8 * 16; e += 32) *(uint32_t*)(xq + (e >> 4) * NB * 64 + t * 64 + (e & 15) * 4) = 0u;
      __syncwarp();
      F[t] = 0, T[t] = 0;
    }
  }
}
template <int NB>
__device__ __forceinline__ void poll_tokens(const InSpec& in, int c0, int t0, int batch, uint32_t epoch, int lane,
                                            float (&u)[2][2][4]) {
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (t0 + i < batch) {
        const InSpec it = token_of(in, t0 + i);
        ok &= load_group(it, c0 + 4 * lane, epoch, u[i][0]);
        ok &= load_group(it, c0 + 4 * (lane + 32), epoch, u[i][1]);
      }
    }
    if (__all_sync(0xffffffffu, ok)) break;
    if (kPollSleepNs) __nanosleep(kPollSleepNs);
  }
}

template <int NB>
__device__ __forceinline__ void quantize_chunk_tokens(const InSpec& in, int c, uint32_t epoch, uint8_t* xq, int batch,
                                                      int (&F)[NB], int (&T)[NB], int64_t* dbg = nullptr) {
  const int lane = threadIdx.x & 31;
  const int c0 = c * kChunkCols;
  float sc[2][4];
  // fp16 scales: raw bits before the first poll, converted after it (see quantize_chunk)
  const bool raw_sc = in.iscale && in.sdt == DBF_F16 && c0 + 4 * (lane + 32) + 3 < in.cols;
  uint2 sr0 = make_uint2(0, 0), sr1 = make_uint2(0, 0);
  if (raw_sc) {
    sr0 = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * lane));
    sr1 = __ldg((const uint2*)((const __half*)in.iscale + c0 + 4 * (lane + 32)));
  } else {
    load_scale4(in, c0 + 4 * lane, sc[0]);
    load_scale4(in, c0 + 4 * (lane + 32), sc[1]);
  }
  if (dbg && lane == 0) dbg[0] = gtimer();
  float u[2][2][4];
  poll_tokens<NB>(in, c0, 0, batch, epoch, lane, u);  // tokens 0, 1
  if (raw_sc) {
    const float2 a0 = __half22float2(*(const __half2*)&sr0.x), b0 = __half22float2(*(const __half2*)&sr0.y);
    const float2 a1 = __half22float2(*(const __half2*)&sr1.x), b1 = __half22float2(*(const __half2*)&sr1.y);
    sc[0][0] = a0.x, sc[0][1] = a0.y, sc[0][2] = b0.x, sc[0][3] = b0.y;
    sc[1][0] = a1.x, sc[1][1] = a1.y, sc[1][2] = b1.x, sc[1][3] = b1.y;
  }
  if constexpr (NB > 2) {
    // tokens 2, 3 of an LL input: their words are loaded now and stay in flight while tokens 0, 1
    // are quantized (a second poll only if they were not all current)
    uint4 v[2][2];
    const bool ll = in.kind == 1;
    if (ll) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (2 + i < batch) {
          const uint32_t* x = (const uint32_t*)token_of(in, 2 + i).x;
          v[i][0] = ld_ll16x4(x + c0 + 4 * lane);
          v[i][1] = ld_ll16x4(x + c0 + 4 * (lane + 32));
        }
      }
    }
    if (dbg && lane == 0) dbg[1] = gtimer();
    emit_tokens<NB>(u, sc, xq, 0, batch, lane, F, T);
    if (dbg && lane == 0) dbg[3] = gtimer();
    bool ok = ll;
    if (ll) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (2 + i < batch) {
          ok &= ll_group(v[i][0], c0 + 4 * lane, in.cols, epoch, u[i][0]);
          ok &= ll_group(v[i][1], c0 + 4 * (lane + 32), in.cols, epoch, u[i][1]);
        }
      }
    }
    if (!__all_sync(0xffffffffu, ok)) poll_tokens<NB>(in, c0, 2, batch, epoch, lane, u);
    if (dbg && lane == 0) dbg[4] = gtimer();
    emit_tokens<NB>(u, sc, xq, 2, batch, lane, F, T);
    if (dbg && lane == 0) dbg[6] = gtimer();
  } else {
    emit_tokens<NB>(u, sc, xq, 0, batch, lane, F, T);
  }
}

// The producer lane: stream each run's packed signs (contiguous in HBM) and its 128-byte record into
// the shared-memory ring with cp.async.bulk, L2 evict_first.  Every piece of a run completes on the
// FIRST slot's full barrier (armed once with the run's total bytes), so the compute warps wait on
// one barrier per run.  It never waits on activations: later layers stream while a stage waits.
__device__ __forceinline__ void stream_runs(const dbf_engine_run* R, int r0, int r1, uint8_t* ring,
                                            dbf_engine_run* hdr, uint64_t* full, uint64_t* empty,
                                            int ring_slots, const volatile int* run_now = nullptr) {
  const uint64_t pol = evict_first_policy();
  int slot = 0;
  uint32_t phase = 0;
  const void* n_tiled = nullptr;
  int n_cols = 1, n_units = 0;
  if (r0 < r1) { n_tiled = R[r0].tiled; n_cols = R[r0].cols; n_units = R[r0].nunits; }
  for (int i = r0; i < r1; ++i) {
    const uint8_t* src = (const uint8_t*)n_tiled;
    const int cols = n_cols, nunits = n_units;
    if (i + 1 < r1) { n_tiled = R[i + 1].tiled; n_cols = R[i + 1].cols; n_units = R[i + 1].nunits; }
    const int total = nunits * ((cols + kChunkCols - 1) / kChunkCols) * kChunkBytes;
    int slot0 = slot;
    for (int off = 0; off < total; off += kSlotBytes) {
      const int n = min(kSlotBytes, total - off);
      mbar_wait(&empty[slot], phase ^ 1u);
      if (off == 0) {
        slot0 = slot;
        mbar_arrive_expect_tx(&full[slot0], total + (int)sizeof(dbf_engine_run));
        bulk_g2s(&hdr[slot0], R + i, sizeof(dbf_engine_run), &full[slot0], pol);
      }
      bulk_g2s(ring + (size_t)slot * kSlotBytes, src + off, n, &full[slot0], pol);
      // pacing: pieces of runs more than kPaceAhead runs ahead of the compute warps are spaced
      // kPaceNs apart, so a burst of prefetch (a run's slots freed at once) does not queue in
      // front of the LL handoff loads of the stage in progress (7B step -4 %, measured with
      // 300-2000 ns; runs that are needed next are streamed at full speed)
      if (kPaceNs && (!run_now || i - r0 > *run_now + kPaceAhead)) __nanosleep(kPaceNs);
      if (++slot == ring_slots) { slot = 0; phase ^= 1u; }
    }
  }
}

// Fused one-shot all-reduce (dbf_engine_program.ar_*), once per CTA after its last run: every
// finalize already pushed this rank's partial rows to every peer, so the 16 compute warps meet,
// thread 0 issues ONE system-scope fence and raises the row blocks of the CTA's plain-output runs
// in every peer's flags (a fence per run cost ~10 us per layer: measured), the (row block, rank)
// flags are polled in parallel (20 s watchdog), then y = a * sum over ranks in rank order (fp64,
// rounded once to fp32) -- the same bits on every rank, and the same formula as
// dbf_forward_allreduce's combine (csrc/decode.cu).
struct ArArgs {
  const uint64_t* recv;
  const uint64_t* flags;
  const void* a;
  uint32_t* epoch;
  int world, rank, bt, sdt, ydt;
  int64_t ldy;
  void* y_override;
};

// the kernel's view of dbf_engine_program without the ar_* tail (which travels as a separate,
// trailing kernel parameter, so the plain engine's parameter layout is unchanged)
struct EngineCore {
  const dbf_engine_run* runs;
  const int32_t* cta_offsets;
  uint32_t* run_counter;
  int64_t* trace;
  int32_t nvectors, grid, max_cols, batch;
  const void* x_override;
  void* y_override;
  void* qscratch;
  int64_t qscratch_cta_bytes;
};

struct ArRun {
  void* out_plain;
  int rows, rb, nunits, pad;
};

__device__ __noinline__ void allreduce_cta(const ArArgs ar, const dbf_engine_run* R, int r0, int r1, int batch,
                                           uint32_t ep, ArRun* rs, int rs_cap) {
  asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");  // every push of the CTA issued
  // the CTA's run records, fetched once in parallel into shared memory (rs: the partial-sum area,
  // free now): walking them from global memory one by one cost ~1 us per run and loop (measured)
  const int nr = min(r1 - r0, rs_cap);
  for (int i = threadIdx.x; i < nr; i += kWarps * 32)
    rs[i] = ArRun{R[r0 + i].out_plain, R[r0 + i].rows, R[r0 + i].rb, R[r0 + i].nunits, 0};
  asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
  auto run = [&](int i) -> ArRun {
    return i - r0 < nr ? rs[i - r0] : ArRun{R[i].out_plain, R[i].rows, R[i].rb, R[i].nunits, 0};
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int i = r0; i < r1; ++i) {
      const ArRun r = run(i);
      if (!r.out_plain) continue;
      const int nrb = (r.rows + kRowBlock - 1) / kRowBlock;
      for (int u = 0; u < r.nunits; ++u)
        for (int g2 = 0; g2 < ar.world; ++g2)
          st_relaxed_sys_u32((uint32_t*)ar.flags[g2] + (size_t)ar.rank * nrb + r.rb + u, ep);
    }
  }
  const uint32_t* myflags = (const uint32_t*)ar.flags[ar.rank];
  for (int i = r0; i < r1; ++i) {
    const ArRun r = run(i);
    if (!r.out_plain) continue;
    const int nrb = (r.rows + kRowBlock - 1) / kRowBlock;
    for (int j = threadIdx.x; j < r.nunits * ar.world; j += kWarps * 32) {
      const uint32_t* f = myflags + (size_t)(j % ar.world) * nrb + r.rb + j / ar.world;
      const long long t0 = gtimer();
      // epochs only grow: a peer already on its next call has also pushed this one
      while ((int32_t)(ld_acquire_sys_u32(f) - ep) < 0) {
        __nanosleep(32);
        if (gtimer() - t0 > 20ll * 1000 * 1000 * 1000) __trap();  // 20 s watchdog: a peer is gone
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
  for (int i = r0; i < r1; ++i) {
    const ArRun r = run(i);
    if (!r.out_plain) continue;
    void* y = ar.y_override ? ar.y_override : r.out_plain;
    const int rows = r.rows, rb = r.rb, nunits = r.nunits;
    const float* recv = (const float*)ar.recv[ar.rank] + (size_t)(ep & 1u) * ar.world * ar.bt * rows;
    for (int j = threadIdx.x; j < nunits * 16 * batch; j += kWarps * 32) {
      const int t = (j >> 4) % batch, row = (rb + j / (16 * batch)) * 16 + (j & 15);
      if (row >= rows) continue;
      double acc = 0.0;
      for (int src = 0; src < ar.world; ++src)
        acc += (double)__ldcg(recv + ((size_t)src * ar.bt + t) * rows + row);
      double a = 1.0;
      if (ar.a) {
        switch (ar.sdt) {
          case DBF_F16: a = (double)__half2float(((const __half*)ar.a)[row]); break;
          case DBF_F32: a = (double)((const float*)ar.a)[row]; break;
          case DBF_F64: a = ((const double*)ar.a)[row]; break;
          default: a = (double)__bfloat162float(((const __nv_bfloat16*)ar.a)[row]); break;
        }
      }
      const double v = (double)(float)acc * a;
      const int64_t o = (int64_t)t * ar.ldy + row;
      switch (ar.ydt) {
        case DBF_F16: ((__half*)y)[o] = __float2half_rn((float)v); break;
        case DBF_F32: ((float*)y)[o] = (float)v; break;
        case DBF_F64: ((double*)y)[o] = v; break;
        default: ((__nv_bfloat16*)y)[o] = __float2bfloat16_rn((float)v); break;
      }
    }
  }
}

// The MMAs of units u0 and u0 + 1 (has1) against chunk c of the run (signs resident in the ring),
// as the two units' exact chunk sums P = s/4 - T (as floats) v[unit][row g / g + 8] of this lane's
// token; the caller accumulates acc = fma(P, 1 / (2^F kQScale), acc) with an explicit FMA (left
// to the compiler, the multiply-add was contracted in some unrolled positions and not in others,
// so a unit's sum depended on its place in a run, i.e. on the grid).
__device__ __forceinline__ void pair_mma(const uint8_t* ring, int ring_slots, int slot0, int nch, int c, int u0,
                                         bool has1, const uint2 (&b)[8], int Tt, int lane,
                                         float (&v)[2][2]) {
        uint4 w[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int off = ((u0 + (h && has1 ? 1 : 0)) * nch + c) * kChunkBytes;
          int slot = slot0 + (off >> 14);
          if (slot >= ring_slots) slot -= ring_slots;
          w[h] = *((const uint4*)(ring + (size_t)slot * kSlotBytes + (off & (kSlotBytes - 1))) + lane);
        }
        int ac[2][DBF_CHAINS][4] = {};  // per unit: independent accumulator chains
        if (has1) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          // k-block r = 4s + t reads (word >> 4s) & (0x01010101 << t): A bytes 2^t * bit
          const uint32_t m = 0x01010101u << (r & 3);
          const int sh = 4 * (r >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            imma(ac[h][r % DBF_CHAINS], (w[h].x >> sh) & m, (w[h].y >> sh) & m, (w[h].z >> sh) & m, (w[h].w >> sh) & m,
                 b[r].x, b[r].y);
        }
        } else {  // odd last unit: one MMA stream (its pair partner would be discarded)
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint32_t m = 0x01010101u << (r & 3);
            const int sh = 4 * (r >> 2);
            // the idle second unit's accumulators carry a second chain (half the dependent MMA
            // latency: single-unit runs are the widest segments' case)
            imma(ac[r & 1][0], (w[0].x >> sh) & m, (w[0].y >> sh) & m, (w[0].z >> sh) & m, (w[0].w >> sh) & m,
                 b[r].x, b[r].y);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) ac[0][0][e] += ac[1][0][e];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // columns 2*tig, 2*tig+1 (token tig's digit planes) of rows g, g+8: s = 8 * sum bit X
          int s0 = ac[h][0][0], s1 = ac[h][0][1], s2 = ac[h][0][2], s3 = ac[h][0][3];
#pragma unroll
          for (int q = 1; q < DBF_CHAINS; ++q) s0 += ac[h][q][0], s1 += ac[h][q][1], s2 += ac[h][q][2], s3 += ac[h][q][3];
          v[h][0] = (float)(((s0 + 256 * s1) >> 2) - Tt);  // exact (|P| < 2^24)
          v[h][1] = (float)(((s2 + 256 * s3) >> 2) - Tt);
        }
}

// pair_mma with the two units' chunk addresses already resolved (the caller walks them through the
// ring incrementally: the unit-pair-outer mode's per-chunk address arithmetic, ~16 instructions per
// 16 IMMAs, was the bulk of its loop overhead at 70B widths; 70B 16 blocks 1597 -> 1579 us)
__device__ __forceinline__ void pair_mma_p(const uint4* p0, const uint4* p1, bool has1, const uint2 (&b)[8],
                                           int Tt, float (&v)[2][2]) {
        uint4 w[2];
        w[0] = *p0;
        w[1] = *p1;
        int ac[2][DBF_CHAINS][4] = {};
        if (has1) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint32_t m = 0x01010101u << (r & 3);
          const int sh = 4 * (r >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            imma(ac[h][r % DBF_CHAINS], (w[h].x >> sh) & m, (w[h].y >> sh) & m, (w[h].z >> sh) & m, (w[h].w >> sh) & m,
                 b[r].x, b[r].y);
        }
        } else {
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint32_t m = 0x01010101u << (r & 3);
            const int sh = 4 * (r >> 2);
            imma(ac[r & 1][0], (w[0].x >> sh) & m, (w[0].y >> sh) & m, (w[0].z >> sh) & m, (w[0].w >> sh) & m,
                 b[r].x, b[r].y);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) ac[0][0][e] += ac[1][0][e];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int s0 = ac[h][0][0], s1 = ac[h][0][1], s2 = ac[h][0][2], s3 = ac[h][0][3];
#pragma unroll
          for (int q = 1; q < DBF_CHAINS; ++q) s0 += ac[h][q][0], s1 += ac[h][q][1], s2 += ac[h][q][2], s3 += ac[h][q][3];
          v[h][0] = (float)(((s0 + 256 * s1) >> 2) - Tt);
          v[h][1] = (float)(((s2 + 256 * s3) >> 2) - Tt);
        }
}

// AR: the program's last stage carries the fused all-reduce (dbf_engine_program.ar_*); a separate
// instantiation, so the plain engine carries none of its code (measured +1.3-7 % when shared)
template <int NB, int XS, bool AR>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(EngineCore prog, int ring_slots, ArArgs ar) {
  constexpr int kMaxUnits = max_units<NB>();
  constexpr int kChunkQ = kChunkQBytes1 * NB, kPartFloats = kWarps * kMaxUnits * 16 * NB;
  // quantized chunks kept per warp (xs_chunks_of: sized by the program's widest input at batch 1)
  constexpr int xsc = XS;
  constexpr int xsb = xsc * kChunkQ;
  extern __shared__ __align__(128) uint8_t smem[];
  Smem sm;
  sm.ring = smem;
  sm.hdr = (dbf_engine_run*)(sm.ring + (size_t)ring_slots * kSlotBytes);
  sm.xs = (uint8_t*)(sm.hdr + ring_slots);
  sm.part = (float*)(sm.xs + kWarps * xsb);
  sm.full = (uint64_t*)(sm.part + 2 * kPartFloats);
  sm.empty = sm.full + ring_slots;
  // rarely-read per-warp / per-CTA scalars live in shared memory, not in (spilled) registers:
  // the quantized chunks' F and T for reuse across runs, the launch's epoch base, and each
  // warp's ring cursor {next first slot, full-barrier parities}
  int* qft = (int*)(sm.empty + ring_slots);  // [kWarps][xs_chunks][NB][2]
  uint32_t* ep_base_s = (uint32_t*)(qft + kWarps * xsc * NB * 2);
  // input key (vector, input scale) of the quantized chunks, double-buffered by run parity: run j
  // reads slot (j+1)&1 (written by warp 0 during run j-1, before that run's barrier) and writes j&1
  struct InKey { const void* iscale; int vec; int pad; };
  InKey* inkey = (InKey*)(ep_base_s + 4);
  int2* cursor = (int2*)(inkey + 2);  // [kWarps]
  // the run's output fields live in shared memory (double-buffered by run parity, written by warp
  // 0 at run start) instead of registers held across the MMA loop: 4 tokens 48 -> 8 bytes of
  // spills (7B 2531 -> 2292 us), 1 token 1042 -> 1027 us; 2 tokens measured 1.6 % slower, kept off
  constexpr bool kRunOutSmem = NB != 2;
  struct RunOut { void* out_plain; uint32_t* ll_out; int rows, rb, odt; uint32_t ep_out; };
  RunOut* runout = (RunOut*)(cursor + kWarps);  // [2]
  volatile int* run_now = (volatile int*)(runout + 2);  // the compute warps' current run (producer pacing)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring_slots; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int r0 = prog.cta_offsets[blockIdx.x], r1 = prog.cta_offsets[blockIdx.x + 1];
  if (threadIdx.x == 0) {
    *ep_base_s = *prog.run_counter;  // (launches * nvectors) mod 65535, advanced below
    if (AR) ep_base_s[1] = *ar.epoch + 1u;  // this call's all-reduce epoch
    *run_now = 0;
    inkey[0].vec = inkey[1].vec = -1;
    inkey[0].iscale = inkey[1].iscale = nullptr;
  }
  __syncthreads();
  const dbf_engine_run* R = prog.runs;

  if (warp >= kProdWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
    // ---------------- producer: stream each run's packed signs (contiguous) into the ring -----
    if (warp == kProdWarp && lane == 0)
      stream_runs(R, r0, r1, sm.ring, sm.hdr, sm.full, sm.empty, ring_slots, run_now);
    return;
  }

  // ---------------- compute warps -------------------------------------------------------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kComputeRegs));
  const int g = lane >> 2, tig = lane & 3;
  const int batch = prog.batch < 1 ? 1 : prog.batch;  // tokens present (<= NB)
  uint8_t* xs = sm.xs + warp * xsb;
  // this lane's B fragment in a k-block: column g = 2*token + plane (columns >= 2*NB mirror)
  const int xlane = ((lane >> 2) % (2 * NB)) * 32 + (lane & 3) * 8;
  // the quantized chunks stay valid for the next run when it reads the same vector with the same
  // input scale (a stage's units split over several runs of one CTA)
  int* wq = qft + warp * xsc * NB * 2;  // this warp's [xs_chunks][NB][F, T]
  if (lane == 0) cursor[warp] = make_int2(0, 0);  // {first slot of the next run, full parities}
  __syncwarp();
  for (int i = r0; i < r1; ++i) {
    const int j = i - r0, buf = j & 1;
    int64_t* tr = prog.trace ? prog.trace + 4 * (size_t)i : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();
#ifdef DBF_ENGINE_WARP_TRACE
    // debug build only: per (run, warp) stamps [start, pieces, quantized x3, computed x3, barrier, final,
    // first chunk: poll start, poll success, poll count]
    int64_t* wt = prog.trace ? prog.trace + 4 * (size_t)prog.cta_offsets[gridDim.x] + ((size_t)i * kWarps + warp) * 17
                             : nullptr;
#define WT(k) do { if (wt && lane == 0) wt[k] = gtimer(); } while (0)
#else
#define WT(k) do { } while (0)
#endif
    if (warp == 0 && lane == 0) *run_now = j;
    const int2 cur = cursor[warp];
    const int slot0 = cur.x;
    mbar_wait(&sm.full[slot0], ((uint32_t)cur.y >> slot0) & 1u);  // the run's record and ALL its pieces
    WT(0);
    const dbf_engine_run& H = sm.hdr[slot0];
    const int cols = H.cols, nunits = H.nunits;
    InSpec in;
    in.x = (H.in_vec == 0 && prog.x_override) ? prog.x_override : H.x;
    in.iscale = H.iscale;
    in.kind = H.in_kind;
    in.dtype = H.in_dtype;
    in.sdt = H.scale_dtype;
    in.cols = cols;
    in.tstride = in.kind == 1 ? (int64_t)((cols + kChunkCols - 1) / kChunkCols) * kChunkCols : cols;
    // finalize fields (the record's ring slot is recycled once the run is released)
    const int rows = H.rows, rb = H.rb, odt = H.out_dtype;
    const void* oscale = H.oscale;
    void* out_plain = (H.out_plain && prog.y_override) ? prog.y_override : H.out_plain;
    uint32_t* ll_out = (uint32_t*)H.ll_out;
    const uint32_t ep_out = epoch16(*ep_base_s, H.out_vec);
    const int nch = (cols + kChunkCols - 1) / kChunkCols;
    const int npieces = (nunits * nch * kChunkBytes + kSlotBytes - 1) / kSlotBytes;
    const uint32_t ep_in = H.in_kind == 1 ? epoch16(*ep_base_s, H.in_vec) : 0u;
    if constexpr (kRunOutSmem) {
      if (warp == 0 && lane == 0) runout[buf] = RunOut{out_plain, ll_out, rows, rb, odt, ep_out};
    }
    // batch 1: the next run's ring cursor is stored now, so nothing of it stays live across the
    // MMA loop (7B step 1024 -> 1017 us, 70B -3 %); 4 tokens measured 1 % slower, they store it at
    // the end of the run
    if (NB == 1 && lane == 0) {
      int nx = slot0 + npieces;
      if (nx >= ring_slots) nx -= ring_slots;
      cursor[warp] = make_int2(nx, cur.y ^ (1 << slot0));
    }
    float acc0[kMaxUnits], acc1[kMaxUnits];  // rows g, g+8 of each unit for token tig (tig < NB)
#pragma unroll
    for (int u = 0; u < kMaxUnits; ++u) acc0[u] = acc1[u] = 0.f;
    // all of the run's signs are resident before the MMA loop (no waits inside it, so the
    // compiler can interleave the units' loads and MMAs)
    WT(1);
    // the output scale is fetched now as RAW bits and converted only in the finalize: converting
    // here would stall the finalizing warps for a full L2 round trip before their first poll
    // warp 15 - i finalizes item i = (unit fu, token pair fpair) (warps 15, 14, ...: they own the
    // fewest chunks when a run's chunks do not divide by 16); 4 tokens = 2 pairs per unit, so the
    // 16 warps cover 8 units in one pass
    constexpr int kPairs = (NB + 1) / 2;
    const int fu = (kWarps - 1 - warp) / kPairs, fpair = (kWarps - 1 - warp) % kPairs;
    uint32_t osc_bits = in.sdt == DBF_F16 ? 0x3C00u : 0x3F800000u;  // 1.0
    if (oscale && fu < nunits && lane < 16 && (rb + fu) * 16 + lane < rows) {
      const int r = (rb + fu) * 16 + lane;
      osc_bits = in.sdt == DBF_F16 ? (uint32_t)ld_nc_u16((const unsigned short*)oscale + r)
                                   : ld_nc_u32((const uint32_t*)oscale + r);
    }
    constexpr int kReuseChunks = xsc * kWarps;
    const InKey prev = inkey[buf ^ 1];
    // inputs wider than the shared-memory store (batches of 2-4 tokens on wide layers) keep their
    // quantized chunks in the CTA's L2-resident scratch instead: a later run on the same input
    // copies them back rather than polling and quantizing again
    uint8_t* qscr = (NB > 1 && prog.qscratch && nch > kReuseChunks)
                        ? (uint8_t*)prog.qscratch + (size_t)blockIdx.x * prog.qscratch_cta_bytes
                        : nullptr;
    const bool same_in = H.in_vec == prev.vec && in.iscale == prev.iscale;
    const bool reuse = same_in && nch <= kReuseChunks;
    const bool greuse = same_in && qscr != nullptr;
    if (warp == 0 && lane == 0) {
      inkey[buf].vec = (nch <= kReuseChunks || qscr) ? H.in_vec : -1;
      inkey[buf].iscale = in.iscale;
    }
    bool first = true;
    ChunkFetch nf;
    bool fetched = false;
    if constexpr (NB == 1) {
      // the first owned chunk's LL words are requested right away, ahead of the loop's setup
      // (the quantizer re-polls only if they were not yet current): 7B step 1060 -> 1041 us
      if (!reuse && in.kind == 1 && warp < nch) {
        fetch_issue(in, warp, lane, nf);
        fetched = true;
      }
    }
    float* part = sm.part + buf * kPartFloats;
    if constexpr (NB == 1 && XS > DBF_XS_CHUNKS1) {
      // batch 1 on wide programs (the 7-chunk store, e.g. 70B): unit pairs outer, the warp's chunks
      // inner -- the first pass quantizes every owned chunk (kept in shared memory: the store
      // covers the widest input), later passes reuse them, and each pair's sums go to shared
      // memory as soon as its pass ends, so only one pair's accumulators are live at a time.
      // Per-unit chunk order is unchanged (bitwise).  70B 16 blocks 1743 -> 1579 us; on 7B
      // (4-chunk store, mostly one chunk per warp) chunk-outer stays 0.6 % faster.
#pragma unroll
      for (int p = 0; p < kMaxUnits / 2; ++p) {
        const int u0 = 2 * p;
        if (u0 >= nunits) break;
        const bool has1 = u0 + 1 < nunits;
        float a0[2] = {0.f, 0.f}, a1[2] = {0.f, 0.f};  // units u0, u0 + 1: rows g, g + 8
        // ring byte positions of this lane's 16 bytes of (unit, chunk c) for both units, advanced by
        // kWarps chunks per iteration and wrapped at the ring's end
        const int ring_bytes = ring_slots * kSlotBytes;
        int pos0 = slot0 * kSlotBytes + (u0 * nch + warp) * kChunkBytes + lane * 16;
        int pos1 = pos0 + (has1 ? nch * kChunkBytes : 0);
        if (pos0 >= ring_bytes) pos0 -= ring_bytes;
        if (pos1 >= ring_bytes) pos1 -= ring_bytes;
        // the store holds every owned chunk (the host admits batch-1 programs up to 16 x xsc chunks
        // wide, dbf_engine_smem_bytes), so slot = the warp's chunk index; later unit pairs read the
        // stored digits (a wrapped slot index or a width guard in this loop cost 2.6 % on 70B)
        int qs = 0;
        for (int c = warp; c < nch; c += kWarps, ++qs) {
          uint8_t* xq = xs + qs * kChunkQ;
          int Ft, Tt;
          if (p > 0 || reuse) {
            Ft = wq[2 * qs], Tt = wq[2 * qs + 1];
          } else {
            if (fetched) {
              quantize_fetched(in, c, ep_in, xq, Ft, Tt, nf);
            } else {
              quantize_chunk(in, c, ep_in, xq, 64, Ft, Tt);
            }
            if (lane == 0) wq[2 * qs] = Ft, wq[2 * qs + 1] = Tt;
            fetched = in.kind == 1 && c + kWarps < nch;
            if (fetched) fetch_issue(in, c + kWarps, lane, nf);
            if (tr && first && warp == 0 && lane == 0) tr[1] = gtimer();
            if (first) WT(2);  // (trace build) first owned chunk quantized
            first = false;
          }
          uint2 b[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) b[r] = *(const uint2*)(xq + r * 64 + xlane);
          const float inv = __int_as_float((127 - Ft) << 23) * kQInv;
          float v[2][2];
          pair_mma_p((const uint4*)(sm.ring + pos0), (const uint4*)(sm.ring + pos1), has1, b, Tt, v);
          pos0 += kWarps * kChunkBytes;
          pos1 += kWarps * kChunkBytes;
          if (pos0 >= ring_bytes) pos0 -= ring_bytes;
          if (pos1 >= ring_bytes) pos1 -= ring_bytes;
          a0[0] = __fmaf_rn(v[0][0], inv, a0[0]);
          a1[0] = __fmaf_rn(v[0][1], inv, a1[0]);
          a0[1] = __fmaf_rn(v[1][0], inv, a0[1]);
          a1[1] = __fmaf_rn(v[1][1], inv, a1[1]);
        }
        if (tig == 0) {
          float* pu = part + (warp * kMaxUnits + u0) * 16;
          pu[g] = a0[0];
          pu[g + 8] = a1[0];
          if (has1) {
            pu[16 + g] = a0[1];
            pu[16 + g + 8] = a1[1];
          }
        }
        if (p < 3) WT(5 + p);  // (trace build) unit pair p computed
      }
      if (tr && warp == 0 && lane == 0) tr[2] = gtimer();
    } else {
    for (int c = warp; c < nch; c += kWarps) {
        const int qs = (c / kWarps) % xsc;
        uint8_t* xq = xs + qs * kChunkQ;
        // the chunk exponent F and quantized sum T of this lane's token tig (lanes tig >= NB hold
        // mirrored columns that are discarded); every token's pair is kept in shared memory (wq)
        // for reuse by the next run, and for NB > 1 the lanes pick theirs up from there
        int Ft, Tt;
        if constexpr (NB == 1) {
          if (reuse) {
            Ft = wq[2 * qs], Tt = wq[2 * qs + 1];
          } else {
#ifdef DBF_LL_TRACE  // debug build: [4 nruns][nvectors x 2048 publish stamps][nruns x 16 x (start, arrival)]
            int64_t* llt = prog.trace ? prog.trace + 4 * (size_t)prog.cta_offsets[gridDim.x] +
                                             (size_t)prog.nvectors * 2048 + ((size_t)i * kWarps + warp) * 2
                                      : nullptr;
            if (llt && lane == 0 && c == warp) llt[0] = gtimer();
#endif
            if (fetched) {
              quantize_fetched(in, c, ep_in, xq, Ft, Tt, nf);
            } else {
  #ifdef DBF_ENGINE_WARP_TRACE
              quantize_chunk(in, c, ep_in, xq, 64, Ft, Tt, (wt && c == warp) ? wt + 10 : nullptr);
  #else
              quantize_chunk(in, c, ep_in, xq, 64, Ft, Tt);
  #endif
            }
            if (lane == 0) wq[2 * qs] = Ft, wq[2 * qs + 1] = Tt;
#ifdef DBF_LL_TRACE
            if (llt && lane == 0 && c == warp) llt[1] = gtimer();
#endif
            fetched = in.kind == 1 && c + kWarps < nch;
            if (fetched) fetch_issue(in, c + kWarps, lane, nf);
          }
        } else {
          // scratch slot of chunk c: the digits (kChunkQ bytes) then F, T per token (NB * 8 bytes)
          uint8_t* qsc = qscr ? qscr + (size_t)c * (kChunkQ + kQScrFT) : nullptr;
          if (greuse) {  // copy the chunk back from L2 (each lane its own digit bytes; lanes < 2 NB the F, T)
            const uint4* src = (const uint4*)qsc + lane * (kChunkQ / 512);
            uint4 d[kChunkQ / 512];
  #pragma unroll
            for (int i = 0; i < kChunkQ / 512; ++i) d[i] = __ldcg(src + i);
            const int ft = lane < 2 * NB ? __ldcg((const int*)(qsc + kChunkQ) + lane) : 0;
  #pragma unroll
            for (int i = 0; i < kChunkQ / 512; ++i) ((uint4*)xq)[lane * (kChunkQ / 512) + i] = d[i];
            if (lane < 2 * NB) wq[qs * NB * 2 + lane] = ft;
            __syncwarp();
          } else if (!reuse) {
            int F[NB], T[NB];
  #ifdef DBF_ENGINE_WARP_TRACE
            quantize_chunk_tokens<NB>(in, c, ep_in, xq, batch, F, T, (wt && c == warp) ? wt + 10 : nullptr);
  #else
            quantize_chunk_tokens<NB>(in, c, ep_in, xq, batch, F, T);
  #endif
  #pragma unroll
            for (int t = 0; t < NB; ++t)
              if (lane == 0) wq[(qs * NB + t) * 2] = F[t], wq[(qs * NB + t) * 2 + 1] = T[t];
            __syncwarp();
            if (qsc) {  // keep it for the stage's later runs
              uint4* dst = (uint4*)qsc + lane * (kChunkQ / 512);
  #pragma unroll
              for (int i = 0; i < kChunkQ / 512; ++i) __stcg(dst + i, ((const uint4*)xq)[lane * (kChunkQ / 512) + i]);
              if (lane < 2 * NB) __stcg((int*)(qsc + kChunkQ) + lane, wq[qs * NB * 2 + lane]);
            }
          }
          const int2 ftt = *(const int2*)(wq + (qs * NB + (tig < NB ? tig : 0)) * 2);
          Ft = ftt.x, Tt = ftt.y;
        }
        if (tr && first && warp == 0 && lane == 0) tr[1] = gtimer();
        { const int jj = c / kWarps; if (jj < 3) WT(2 + jj); }
        uint2 b[8];
  #pragma unroll
        for (int r = 0; r < 8; ++r) b[r] = *(const uint2*)(xq + r * NB * 64 + xlane);
        const float inv = __int_as_float((127 - Ft) << 23) * kQInv;  // 1 / (2^F * kQScale)
        // units in pairs: two independent MMA streams per warp (the second repeats the last unit
        // when nunits is odd and is then discarded)
  #pragma unroll
        for (int p = 0; p < kMaxUnits / 2; ++p) {
          const int u0 = 2 * p;
          if (u0 >= nunits) break;
          const bool has1 = u0 + 1 < nunits;
          float v[2][2];
          pair_mma(sm.ring, ring_slots, slot0, nch, c, u0, has1, b, Tt, lane, v);
          acc0[u0] = __fmaf_rn(v[0][0], inv, acc0[u0]);
          acc1[u0] = __fmaf_rn(v[0][1], inv, acc1[u0]);
          if (u0 + 1 < kMaxUnits && has1) {
            acc0[u0 + 1] = __fmaf_rn(v[1][0], inv, acc0[u0 + 1]);
            acc1[u0 + 1] = __fmaf_rn(v[1][1], inv, acc1[u0 + 1]);
          }
        }
        { const int jj = c / kWarps; if (jj < 3) WT(5 + jj); }
        first = false;
      }
      if (tr && warp == 0 && lane == 0) tr[2] = gtimer();
      // partials -> shared memory (double-buffered by run parity), then the compute warps meet once
      if (tig < NB) {
  #pragma unroll
        for (int u = 0; u < kMaxUnits; ++u) {
          if (u < nunits) {
            float* pu = part + ((warp * kMaxUnits + u) * NB + tig) * 16;
            pu[g] = acc0[u];
            pu[g + 8] = acc1[u];
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    WT(8);
    if (warp == 0 && lane == 0)  // every compute warp is done with the run's signs
      for (int p = 0; p < npieces; ++p) {
        int sl = slot0 + p;
        if (sl >= ring_slots) sl -= ring_slots;
        mbar_arrive(&sm.empty[sl]);
      }
    // warp 15 - u finalizes unit u: sum the 16 warps' partials in warp order (deterministic), scale,
    // publish; lanes 0-15 / 16-31 take one token each per pass
    const uint32_t osc_raw = __shfl_sync(0xffffffffu, osc_bits, lane & 15);
    const float osc_row = in.sdt == DBF_F16 ? __half2float(__ushort_as_half((unsigned short)osc_raw))
                                            : __uint_as_float(osc_raw);
    if (fu < nunits) {
      RunOut ro;
      if constexpr (kRunOutSmem) ro = runout[buf];
      else ro = RunOut{out_plain, ll_out, rows, rb, odt, ep_out};
      const int row = (ro.rb + fu) * 16 + (lane & 15);
      {
        const int t = 2 * fpair + (lane >> 4);
        if (t < NB && t < batch && row < ro.rows) {
          float v = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < kWarps; ++w2) v += part[((w2 * kMaxUnits + fu) * NB + t) * 16 + (lane & 15)];
          v *= osc_row;
          const __half h = __float2half_rn(v);
          // status: a NaN / inf output (from a non-finite input) or an fp16 overflow of a value
          // that is published in fp16 (LL handoff or fp16 plain output); rare, so one atomic
          const int64_t ll_stride = (int64_t)((ro.rows + kChunkCols - 1) / kChunkCols) * kChunkCols;
          if (ro.ll_out) st_ll16(ro.ll_out + t * ll_stride + row, h, ro.ep_out);
#ifdef DBF_LL_TRACE
          if (prog.trace && ro.ll_out && (lane & 15) == 0 && t == 0) {
            const dbf_engine_run& H2 = sm.hdr[0];  // unused: out_vec comes from the run record below
            (void)H2;
            prog.trace[4 * (size_t)prog.cta_offsets[gridDim.x] + (size_t)R[i].out_vec * 2048 + ro.rb + fu] = gtimer();
          }
#endif
          if (ro.out_plain) {
            if (AR && ar.world == 1) {
              // world 1: the combine's formula in place (same bits, no fence / flags / poll)
              double a = 1.0;
              if (ar.a) {
                switch (ar.sdt) {
                  case DBF_F16: a = (double)__half2float(((const __half*)ar.a)[row]); break;
                  case DBF_F32: a = (double)((const float*)ar.a)[row]; break;
                  case DBF_F64: a = ((const double*)ar.a)[row]; break;
                  default: a = (double)__bfloat162float(((const __nv_bfloat16*)ar.a)[row]); break;
                }
              }
              const double yv = (double)v * a;
              void* y = ar.y_override ? ar.y_override : ro.out_plain;
              const int64_t o = (int64_t)t * ar.ldy + row;
              switch (ar.ydt) {
                case DBF_F16: ((__half*)y)[o] = __float2half_rn((float)yv); break;
                case DBF_F32: ((float*)y)[o] = (float)yv; break;
                case DBF_F64: ((double*)y)[o] = yv; break;
                default: ((__nv_bfloat16*)y)[o] = __float2bfloat16_rn((float)yv); break;
              }
            } else if (AR) {
              // fused all-reduce, push half: the unrounded fp32 partial into slot ar_rank of every
              // peer's receive buffer (NVLink P2P stores through the mapped peer addresses)
              const size_t idx = (size_t)(ep_base_s[1] & 1u) * ar.world * ar.bt * ro.rows +
                                 ((size_t)ar.rank * ar.bt + t) * ro.rows + row;
              for (int g2 = 0; g2 < ar.world; ++g2) ((float*)ar.recv[g2])[idx] = v;
            } else if (ro.odt == DBF_F16) {
              ((__half*)ro.out_plain)[(int64_t)t * ro.rows + row] = h;
            } else {
              ((float*)ro.out_plain)[(int64_t)t * ro.rows + row] = v;  // fp32 output: unrounded
            }
          }
          // status (after the stores: the publish is on every stage's critical path): a NaN / inf
          // output (from a non-finite input) or an fp16 overflow of a value published in fp16
          if (!(fabsf(v) <= 65504.f) &&
              (!isfinite(v) || ro.ll_out || (ro.out_plain && !AR && ro.odt == DBF_F16)))
            atomicOr(prog.run_counter + 2, isfinite(v) ? kStatusOverflow : kStatusNonFinite);
        }
      }
    }
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
    WT(9);
#undef WT
    if (NB != 1 && lane == 0) {
      int nx = slot0 + npieces;
      if (nx >= ring_slots) nx -= ring_slots;
      cursor[warp] = make_int2(nx, cur.y ^ (1 << slot0));
    }
    __syncwarp();
  }
  if (AR && ar.world > 1)
    allreduce_cta(ar, R, r0, r1, batch, ep_base_s[1], (ArRun*)sm.part,
                  (int)(2 * kPartFloats * sizeof(float) / sizeof(ArRun)));
  // the last CTA to finish advances the launch counter (every CTA read it at its start, and the
  // next launch is stream-ordered after this one): no separate advance kernel per step
  if (warp == 0 && lane == 0 && atomicAdd(prog.run_counter + 1, 1u) == gridDim.x - 1) {
    prog.run_counter[1] = 0u;
    // the epoch base itself advances by nvectors mod 65535 (nvectors % 65535 != 0, checked at
    // launch), so consecutive launches never share an epoch for any vector, however many run
    prog.run_counter[0] = (prog.run_counter[0] + (uint32_t)prog.nvectors) % 65535u;
    if (AR) *ar.epoch += 1u;  // every CTA read it at its start
  }
}

// shared memory besides the per-slot parts (16 KB ring slot + 128 B record + 2 mbarriers)
inline size_t fixed_smem(int nb, int xsc) {
  const int xs = xsc * kChunkQBytes1 * nb;
  return (size_t)kWarps * xs + 2 * (size_t)part_floats(nb) * 4 + (size_t)kWarps * xsc * nb * 2 * 4 + 48 +
         (size_t)kWarps * 8 + 128;
}
constexpr size_t kPerSlot = kSlotBytes + sizeof(dbf_engine_run) + 2 * 8;
inline size_t fixed_smem_of(int nb, int max_cols) { return fixed_smem(nb, xs_chunks_of(nb, max_cols)); }
inline int ring_slots(int nb, int max_cols) {
  return std::min((int)((kMaxSmem - fixed_smem_of(nb, max_cols)) / kPerSlot), kMaxSlots);
}
inline size_t smem_bytes(int slots, int nb, int max_cols) {
  return (size_t)slots * kPerSlot + fixed_smem_of(nb, max_cols);
}
inline int nb_for(int batch) { return batch <= 1 ? 1 : (batch <= 2 ? 2 : 4); }

}  // namespace engine
}  // namespace dbf

using namespace dbf;

static_assert(sizeof(dbf_engine_run) == 128, "run record must be 128 bytes");

extern "C" int dbf_engine_build_runs(const dbf_engine_segment* segments, int32_t nsegments,
                                     const dbf_engine_vector* vectors, int32_t nvectors, const int32_t* runs,
                                     int32_t nruns, int32_t batch, uint32_t* ready, dbf_engine_run* out) {
  if (!segments || !vectors || !runs || !out || nsegments < 1 || nvectors < 1 || nruns < 0)
    return DBF_ERR_INVALID_ARGUMENT;
  // units producing each vector (one segment writes each LL vector)
  std::vector<uint32_t> producers(nvectors, 0);
  int max_cols = 1;
  for (int s = 0; s < nsegments; ++s) max_cols = std::max(max_cols, (int)segments[s].cols);
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
    if (n > engine::max_units_of(engine::nb_for(batch)) ||
        (int64_t)n * chunks(g.cols) * kChunkBytes >
            (int64_t)(engine::ring_slots(engine::nb_for(batch), max_cols) / 2) * engine::kSlotBytes)
      return DBF_ERR_SHAPE;  // split longer runs (dbf_engine_run_limits_cols)
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

#ifdef DBF_LL_TRACE
extern "C" int dbf_debug_ll_rtt(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dbf::engine::g_ll_rtt, 16);
  unsigned long long z[2] = {0, 0};
  cudaMemcpyToSymbol(dbf::engine::g_ll_rtt, z, 16);
  return DBF_OK;
}
#endif

extern "C" int dbf_engine_smem_bytes(int32_t max_cols, int32_t batch, size_t* bytes) {
  if (max_cols < 1 || !bytes || batch < 1 || batch > 4) return DBF_ERR_INVALID_ARGUMENT;
  const int nb = engine::nb_for(batch);
  const int slots = engine::ring_slots(nb, max_cols);
  // one 16-row unit of the widest segment must fit half the ring
  if (slots < engine::kMinSlots || chunks(max_cols) * kChunkBytes > (int64_t)(slots / 2) * engine::kSlotBytes)
    return DBF_ERR_UNSUPPORTED;
  // batch 1 keeps every quantized input chunk of a warp in shared memory (up to 16 x 7 chunks =
  // 28672 columns: the widest Llama-2 input); wider inputs take the batched kernels
  if (nb == 1 && chunks(max_cols) > (int64_t)engine::kWarps * DBF_XS_CHUNKS1_MAX) return DBF_ERR_UNSUPPORTED;
  *bytes = engine::smem_bytes(slots, nb, max_cols);
  return DBF_OK;
}

extern "C" size_t dbf_engine_qscratch_bytes(int32_t max_cols, int32_t batch) {
  if (max_cols < 1 || batch < 2 || batch > 4) return 0;
  const int nb = engine::nb_for(batch);
  const int64_t nch = chunks(max_cols);
  if (nch <= (int64_t)engine::xs_chunks_of(nb, max_cols) * engine::kWarps) return 0;
  return (size_t)nch * (engine::kChunkQBytes1 * nb + engine::kQScrFT);  // per CTA
}

extern "C" int dbf_engine_run_limits_cols(int32_t max_cols, int32_t batch, int32_t* max_units,
                                          int64_t* max_run_bytes) {
  if (!max_units || !max_run_bytes || batch < 1 || batch > 4 || max_cols < 0) return DBF_ERR_INVALID_ARGUMENT;
  *max_units = engine::max_units_of(engine::nb_for(batch));
  // a run's signs stay resident until every compute warp is done with it; leave room to prefetch
  *max_run_bytes = (int64_t)(engine::ring_slots(engine::nb_for(batch), max_cols) / 2) * engine::kSlotBytes;
  return DBF_OK;
}

extern "C" int dbf_engine_run_limits(int32_t batch, int32_t* max_units, int64_t* max_run_bytes) {
  return dbf_engine_run_limits_cols(0, batch, max_units, max_run_bytes);
}

template <typename K>
static int engine_occupancy_of(K kern, size_t smem, int32_t* blocks_per_sm, int32_t* regs_per_thread) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, engine::kMaxSmem);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  *regs_per_thread = fa.numRegs;
  int nb = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, engine::kThreads, smem);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  *blocks_per_sm = nb;
  return DBF_OK;
}

extern "C" int dbf_engine_occupancy(int32_t max_cols, int32_t* blocks_per_sm, int32_t* regs_per_thread) {
  if (!blocks_per_sm || !regs_per_thread || max_cols < 1) return DBF_ERR_INVALID_ARGUMENT;
  size_t smem = 0;
  int st = dbf_engine_smem_bytes(max_cols, 1, &smem);
  if (st != DBF_OK) return st;
  return engine::xs_chunks_of(1, max_cols) == DBF_XS_CHUNKS1
             ? engine_occupancy_of(engine::engine_kernel<1, DBF_XS_CHUNKS1, false>, smem, blocks_per_sm, regs_per_thread)
             : engine_occupancy_of(engine::engine_kernel<1, DBF_XS_CHUNKS1_MAX, false>, smem, blocks_per_sm, regs_per_thread);
}

template <int NB, int XS, bool AR>
static int engine_launch_nb(const dbf_engine_program* program, cudaStream_t s) {
  size_t smem = 0;
  int st = dbf_engine_smem_bytes(program->max_cols, NB, &smem);
  if (st != DBF_OK) return st;
  const int slots = engine::ring_slots(NB, program->max_cols);
  st = ensure_smem_attr<engine::engine_kernel<NB, XS, AR>>(engine::kMaxSmem);
  if (st != DBF_OK) return st;
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
  const dbf_engine_program& p = *program;
  const engine::EngineCore core{p.runs, p.cta_offsets, p.run_counter, p.trace, p.nvectors, p.grid, p.max_cols,
                                p.batch, p.x_override, p.y_override, p.qscratch, p.qscratch_cta_bytes};
  const engine::ArArgs ar{p.ar_recv, p.ar_flags, p.ar_a, p.ar_epoch, p.ar_world, p.ar_rank, p.ar_bt, p.ar_sdt,
                          p.ar_ydt, p.ar_ldy, p.y_override};
  cudaError_t e = cudaLaunchKernelEx(&cfg, engine::engine_kernel<NB, XS, AR>, core, slots, ar);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  return DBF_OK;
}

template <bool AR>
static int engine_launch_ar(const dbf_engine_program* program, cudaStream_t s) {
  const int nb = engine::nb_for(program->batch);
  int st;
  if (nb == 1)
    st = engine::xs_chunks_of(1, program->max_cols) == DBF_XS_CHUNKS1
             ? engine_launch_nb<1, DBF_XS_CHUNKS1, AR>(program, s)
             : engine_launch_nb<1, DBF_XS_CHUNKS1_MAX, AR>(program, s);
  else
    st = nb == 2 ? engine_launch_nb<2, 4, AR>(program, s)
                 : (engine::xs_chunks_of(4, program->max_cols) == 2 ? engine_launch_nb<4, 2, AR>(program, s)
                                                                     : engine_launch_nb<4, 1, AR>(program, s));
  if (st != DBF_OK) return st;
  return check_launch();
}

extern "C" int dbf_engine_launch(const dbf_engine_program* program, void* stream) {
  if (!program || !program->runs || !program->cta_offsets || !program->run_counter || program->grid < 1 ||
      program->max_cols < 1 || program->batch < 1 || program->batch > 4 || program->nvectors < 1 ||
      program->nvectors % 65535 == 0)
    return DBF_ERR_INVALID_ARGUMENT;
  if (program->ar_world &&
      (program->ar_world < 0 || program->ar_world > 64 || program->ar_rank < 0 ||
       program->ar_rank >= program->ar_world || !program->ar_recv || !program->ar_flags || !program->ar_epoch ||
       program->ar_bt < program->batch || program->ar_ldy < 1 || program->ar_ydt < DBF_F16 || program->ar_ydt > DBF_BF16 ||
       (program->ar_a && (program->ar_sdt < DBF_F16 || program->ar_sdt > DBF_BF16))))
    return DBF_ERR_INVALID_ARGUMENT;
  return program->ar_world ? engine_launch_ar<true>(program, (cudaStream_t)stream)
                           : engine_launch_ar<false>(program, (cudaStream_t)stream);
}

