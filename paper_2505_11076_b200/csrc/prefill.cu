// DBF prefill / batched path (>= 64 tokens): the two sign GEMMs of one DBF forward on the
// 5th-generation tensor cores (tcgen05 + TMEM), replacing kernel.forward (kernel.py:48-62) for
// token batches where the layer is a real dense contraction:
//
//   GEMM1  t[T, k] = mid (.) ( X[T, m] . (B (.) b)^T )      B: k x m signs, b folded into B
//   GEMM2  Y[T, n] = a   (.) ( t[T, k] . A^T )              A: n x k signs
//
// One kernel, `sign_gemm_kernel`, runs either GEMM: out[T, rows] = rscale (.) (act . (S (.) kscale)^T)
// with S a rows x K sign matrix in the PAIRED word layout (include/dbf_b200.h, dbf_pair_signs).
//
// Per CTA (sign_gemm_kernel, one output tile per CTA): 128 sign rows (MMA M, TMEM lanes) x 256 tokens
// (MMA N), accumulated in TMEM (256 fp32 columns).
//   warps 0,2,3  TMA producers: 256 x 64 fp16 activation boxes (128-byte swizzle) into a 6-stage smem
//                ring, one issuing lane per stage.
//   warp 1       TMEM allocator + MMA issuer (one thread): tcgen05.mma.kind::f16, M=128 N=256 K=16,
//                A operand (the expanded signs) from TMEM, B operand (activations) from smem.
//   warps 4..11  sign expanders, then epilogue.  Warp w owns TMEM sub-partition w%4 (32 sign rows, one
//                per lane) and word (w-4)/4 of every 64-column K block: per K block a lane turns ONE
//                32-bit word of packed signs into 32 fp16 values +-kscale[c] -- one shift + one LOP3 per
//                fp16 pair, the fp16 sign bit XORed in from the packed bit -- and writes them straight
//                into TMEM with tcgen05.st (32x32b.x16).  The +-1 expansion never touches shared memory
//                or HBM; the activation ring is the only smem traffic of the MMAs.
//   epilogue     16x256b tcgen05.ld of the accumulator, row scale, fp16, stmatrix.trans into the idle
//                ring (128-byte swizzle), two TMA stores.
// Ring stage s couples a smem activation box and a TMEM A slot; both are released by the
// tcgen05.commit of the MMAs that read them.  T <= 256 uses N = the tokens present and splits K.
// sign_layer_kernel (namespace layer, below) runs both GEMMs of a layer as one persistent launch.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include "common.cuh"
#include "sm100.cuh"

namespace dbf {
namespace prefill {

using namespace sm100;

constexpr int UM = 128;          // MMA M (TMEM lanes)
#ifndef DBF_PREFILL_MH
#define DBF_PREFILL_MH 1
#endif
constexpr int MH = DBF_PREFILL_MH;  // M halves per tile (accumulators)
constexpr int BM = MH * UM;      // sign rows per tile
constexpr int BN = 256 / MH;     // tokens per tile (MMA N, accumulator columns)
constexpr int BK = 64;           // K per stage (one 128-byte swizzle atom of fp16)
constexpr int UK = 16;           // K per tcgen05.mma (kind::f16)
#ifndef DBF_PREFILL_STAGES
#define DBF_PREFILL_STAGES 6
#endif
constexpr int STAGES = DBF_PREFILL_STAGES;
constexpr int kAColsPerHalf = BK / 2;         // 32 TMEM columns (2 fp16 per 32-bit column)
constexpr int kAColsPerStage = MH * kAColsPerHalf;
constexpr int kAccCol = 0;                    // accumulator of M half h at column h * BN
constexpr int kTmemCols = 512;
constexpr int kExpWarp0 = 4;
constexpr int kNumProducers = 3;              // warps 0, 2, 3
constexpr int kExpWarps = 8 * MH;
constexpr int kThreads = (kExpWarp0 + kExpWarps) * 32;

struct Params {
  const uint32_t* words;   // rows x pitch PAIRED words
  int64_t pitch;           // words per row
  const __half* kscale;    // K values or nullptr (= 1)
  const __half* rscale;    // rows values or nullptr (= 1)
  __half* out;             // out[tok * ldo + row]
  int64_t ldo;
  int rows, K, T;
  int num_kb;
  long long* trace;        // debug: per-K-block clock64 stamps of CTA (0,0), or nullptr
  // small token counts (T <= 256): the MMA N and the activation box shrink to the tokens present
  // (n_mma, act_bytes), and K may be split over gridDim.z CTAs (kb_per_split K blocks each) that
  // store unscaled fp32 partials part[z][tok][row] for split_reduce_kernel (part == nullptr: no split)
  int n_mma;
  int act_bytes;
  int kb_per_split;
  float* part;
  int tma_out;             // epilogue: fp16 tile staged in shared memory, one TMA store (out_map)
};

template <int NST>
struct __align__(8) BarriersT {
  uint64_t full_act[NST];
  uint64_t full_a[NST];
  uint64_t empty[NST];
  uint64_t acc_full;
  uint32_t tmem_base;
};

// Small-token tiles (T <= kSmallBN): the accumulator needs only kSmallBN TMEM columns, so the ring
// can be twice as deep with 8 KB activation boxes.  At N <= 64 a K block's MMAs take ~128 cycles
// and the 6-stage ring left each K block bound by the activation TMA round trip (~3100 cycles
// over 6 boxes in flight, tools/prefill_trace.py).
constexpr int kSmallBN = 64, kSmallStages = 12;

static_assert(MH * BN + STAGES * kAColsPerStage <= kTmemCols, "TMEM budget (A slots)");
static_assert(MH == 1, "the TMA-store epilogue stages one 128-row accumulator per tile");
static_assert(MH * kSmallBN + kSmallStages * kAColsPerStage <= kTmemCols, "TMEM budget (small tiles)");
template <int TBN, int NST>
inline size_t smem_bytes_for(int num_kb, bool kscale) {
  return 1024 /*align slack*/ + (size_t)NST * TBN * BK * 2 + sizeof(BarriersT<NST>) + 64 + 16 +
         (kscale ? (size_t)num_kb * BK * 2 : 0);
}
inline size_t smem_bytes(int num_kb, bool kscale) { return smem_bytes_for<BN, STAGES>(num_kb, kscale); }

// One paired word (bit q <-> column 2q, bit 16+q <-> column 2q+1 of a 32-column group) -> 16 words of
// fp16 pairs +-ks.  (~w << (15-q)) moves the NEGATED signs of the pair to the fp16 sign positions
// 15 / 31; LOP3 ((x & 0x80008000) ^ ks) applies them.  ks = +1.0 pairs when there is no kscale.
__device__ __forceinline__ void expand_word(uint32_t w, const uint32_t* ks, uint32_t (&v)[16]) {
  const uint32_t nw = ~w;
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = ((nw << (15 - q)) & 0x80008000u) ^ ks[q];
}

template <bool KSCALE, int TBN = BN, int NST = STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    sign_gemm_kernel(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap out_map,
                     const Params p) {
  // tile configuration: the namespace defaults, or the small-token tiles
  constexpr int BN = TBN, STAGES = NST;
  constexpr int kActStageBytes = BN * BK * 2;
  constexpr int kACol0 = MH * BN;
  using Barriers = BarriersT<STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* act = smem;
  Barriers& bar = *reinterpret_cast<Barriers*>(smem + (size_t)STAGES * kActStageBytes);

#ifdef DBF_PREFILL_TRACE
  const long long cta_c0_ = clock64();
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * BM;
  const int tok0 = blockIdx.y * BN;
  const int kb0 = p.part ? (int)blockIdx.z * p.kb_per_split : 0;  // this CTA's K blocks [kb0, kb1)
  const int kb1 = p.part ? min(p.num_kb, kb0 + p.kb_per_split) : p.num_kb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bar.full_act[s], 1);
      mbar_init(&bar.full_a[s], kExpWarps);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&act_map);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&bar.tmem_base);
  // expanders: the first 8 K blocks' sign words and the epilogue's row scales are layer constants,
  // requested before the setup barrier so their HBM latency overlaps it
  uint4 q[4];
  uint32_t ksr[4];      // K scales of the first 8 K blocks (see load_ksr below)
  __half rs_pre[2][2];  // converted where used, so no thread waits for them at the barrier
  // K scales live in registers: for the 8 K blocks of a group, lane L holds in ksr[jp] the fp16 pair
  // (L & 15) of its warp's 32 columns of K block kg + 2 jp + (L >> 4); a K block's 16 pairs are one
  // shuffle each.  (They used to be copied to shared memory before the setup barrier: ~0.8 us on
  // every GEMM1 CTA's critical path, and shared memory a 7th ring stage can use.)
  const int half_w = ((warp - kExpWarp0) >> 2) / MH;
  auto load_ksr = [&](int kg, uint32_t (&r)[4]) {
    const unsigned short* bsrc = reinterpret_cast<const unsigned short*>(p.kscale);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      const int c = (kg + 2 * jp + (lane >> 4)) * BK + half_w * 32 + 2 * (lane & 15);
      r[jp] = !KSCALE ? 0x3C003C00u
                      : ((c < p.K ? (uint32_t)__ldg(bsrc + c) : 0u) | ((c + 1 < p.K ? (uint32_t)__ldg(bsrc + c + 1) : 0u) << 16));
    }
  };
  if (warp >= kExpWarp0) {
    load_ksr(kb0, ksr);
    const int sub = warp & 3, mh = ((warp - kExpWarp0) >> 2) % MH;
    const int grow = row0 + mh * UM + sub * 32 + lane;
    const bool live = grow < p.rows;
    const uint4* wrow = reinterpret_cast<const uint4*>(p.words + (int64_t)(live ? grow : 0) * p.pitch);
    const int nquads = (p.num_kb + 1) >> 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      q[i] = (live && (kb0 >> 1) + i < nquads) ? __ldg(wrow + (kb0 >> 1) + i) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int lb = 0; lb < 2; ++lb)
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int rr = row0 + sub * 32 + lb * 16 + hi * 8 + (lane >> 2);
        rs_pre[lb][hi] = (p.rscale && p.tma_out && rr < p.rows) ? p.rscale[rr] : __float2half(1.f);
      }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  const bool tracing = p.trace && blockIdx.x == 0 && blockIdx.y == 0;
  // programmatic dependent launch: the next kernel on the stream may start its own setup on SMs as
  // they free up; everything that reads the activations or writes the output waits for the
  // previous kernel (griddepcontrol.wait) -- the setup above touches layer constants only
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef DBF_PREFILL_TRACE
  unsigned long long cta_t0 = 0;
  long long* cslot = nullptr;
  {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (p.trace && cta < 4096) cslot = p.trace + 6 * 4096 + 16 * (size_t)cta;
  }
#define CT(i) do { if (cslot) cslot[i] = clock64(); } while (0)
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_t0));
    if (cslot) cslot[4] = cta_c0_;
  }
  if (threadIdx.x == 0) CT(5);
#else
#define CT(i) do { } while (0)
#endif

  if (warp == 0 || warp == 2 || warp == 3) {
    // ---------------- TMA producers ----------------
    // One thread's TMA loads complete one after another (~500 clk per box on B200, measured:
    // tools/microbench/tma.cu), so every ring stage gets its own issuing thread: lanes
    // 0..kPerWarp-1 of the three producer warps (3 issuers for 6 stages left small-token tiles,
    // whose MMAs are short, bound at ~600 cycles per K block).
    constexpr int kPerWarp = (STAGES + kNumProducers - 1) / kNumProducers;
    constexpr int kIssuers = kPerWarp * kNumProducers;
    if (lane < kPerWarp) {
      const int prod = (warp == 0 ? 0 : warp - 1) * kPerWarp + lane;
      const uint64_t pol = policy_evict_last();  // activations are re-read by every row tile
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int kb = kb0 + prod; kb < kb1; kb += kIssuers) {
        const int s = (kb - kb0) % STAGES;
        const uint32_t ph = ((kb - kb0) / STAGES) & 1;
        mbar_wait(&bar.empty[s], ph ^ 1);
        if (tracing) p.trace[5 * p.num_kb + kb] = clock64();
        mbar_arrive_expect_tx(&bar.full_act[s], p.act_bytes);
        tma_load_2d(act + (size_t)s * kActStageBytes, &act_map, kb * BK, tok0, &bar.full_act[s], pol);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_f16_f32(UM, p.n_mma);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int s = (kb - kb0) % STAGES;
        const uint32_t ph = ((kb - kb0) / STAGES) & 1;
        mbar_wait(&bar.full_act[s], ph);
        if (tracing) p.trace[4 * kb + 3] = clock64();
        mbar_wait(&bar.full_a[s], ph);
        tc_fence_after();
        if (tracing) p.trace[4 * p.num_kb + kb] = clock64();
        if (kb == kb0) CT(6);
        const uint32_t a_base = tmem + kACol0 + s * kAColsPerStage;
        const uint32_t b_base = smem_u32(act + (size_t)s * kActStageBytes);
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t bd = sdesc_k_sw128(b_base + kk * UK * 2);
#pragma unroll
          for (int h = 0; h < MH; ++h)
            mma_f16_ts(tmem + kAccCol + h * BN, a_base + h * kAColsPerHalf + kk * (UK / 2), bd, idesc,
                       (kb != kb0) || (kk != 0));
        }
        mma_commit(&bar.empty[s]);
      }
      mma_commit(&bar.acc_full);
      CT(7);
    }
  } else if (warp >= kExpWarp0) {
    // ---------------- sign expanders + epilogue ----------------
    const int sub = warp & 3;                 // TMEM sub-partition this warp may access
    const int mh = ((warp - kExpWarp0) >> 2) % MH;  // M half (accumulator) of this warp's rows
    const int half = ((warp - kExpWarp0) >> 2) / MH;  // which 32-column word of each K block
    const int r = mh * UM + sub * 32 + lane;  // tile row
    const int grow = row0 + r;
    const bool live = grow < p.rows;
    const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
    const uint4* wrow = reinterpret_cast<const uint4*>(p.words + (int64_t)(live ? grow : 0) * p.pitch);
    // one uint4 = words 4i..4i+3 = K blocks 2i (.x/.y) and 2i+1 (.z/.w).  Groups of 8 K blocks
    // (4 quads): the next group's quads are loaded when a group starts, so each load has 8 K blocks
    // of MMA time to arrive (one quad ahead was too short for N = 64 tiles: HBM latency-bound)
    const int nquads = (p.num_kb + 1) >> 1;
    const bool tr = tracing && threadIdx.x == 32 * kExpWarp0;
    for (int kg = kb0; kg < kb1; kg += 8) {  // kb0 is even (splits are whole quads)
      uint4 nq[4];
      uint32_t nksr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int qi = (kg >> 1) + 4 + i;
        nq[i] = (live && qi < nquads && 2 * qi < kb1) ? __ldg(wrow + qi) : make_uint4(0, 0, 0, 0);
      }
      load_ksr(kg + 8, nksr);
#pragma unroll
      // two K blocks per iteration (one slot wait, one tcgen05 store wait and one arrive round per
      // pair): at small token counts the per-K-block bookkeeping bounded the expanders
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        const int kb = kg + 2 * jp;
        if (kb >= kb1) break;
        const bool two = kb + 1 < kb1;
        const int s = (kb - kb0) % STAGES, s1 = (kb + 1 - kb0) % STAGES;
        const uint32_t ph = ((kb - kb0) / STAGES) & 1, ph1 = ((kb + 1 - kb0) / STAGES) & 1;
        uint32_t ks[16], v0[16], v1[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) ks[w] = __shfl_sync(0xffffffffu, ksr[jp], w);
        expand_word(half ? q[jp].y : q[jp].x, ks, v0);
        if (two) {
#pragma unroll
          for (int w = 0; w < 16; ++w) ks[w] = __shfl_sync(0xffffffffu, ksr[jp], 16 + w);
          expand_word(half ? q[jp].w : q[jp].z, ks, v1);
        }
        if (tr) p.trace[4 * kb] = clock64();
        if (lane == 0) {  // one poller per warp
          mbar_wait(&bar.empty[s], ph ^ 1);
          if (two) mbar_wait(&bar.empty[s1], ph1 ^ 1);
        }
        __syncwarp();
        if (tr) p.trace[4 * kb + 1] = clock64();
        tc_fence_after();
        const uint32_t col = tmem + lane_addr + kACol0 + mh * kAColsPerHalf + half * 16;
        tmem_st16(col + s * kAColsPerStage, v0);
        if (two) tmem_st16(col + s1 * kAColsPerStage, v1);
        tmem_wait_st();
        tc_fence_before();
        if (tr) p.trace[4 * kb + 2] = clock64();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bar.full_a[s]);
          if (two) mbar_arrive(&bar.full_a[s1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = nq[i], ksr[i] = nksr[i];
    }
    // epilogue: this warp stores tokens [half*64, half*64+64) of its 32 rows (accumulator mh)
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel may still read the output
    if (lane == 0) mbar_wait(&bar.acc_full, 0);
    if (threadIdx.x == 32 * kExpWarp0) CT(8);
    __syncwarp();
    tc_fence_after();
    const float rs = (live && p.rscale) ? __half2float(p.rscale[grow]) : 1.f;
    if (p.tma_out) {
      // The ring is idle once the accumulator is complete: stage the fp16 tile there in the
      // output's [token][row] layout as two 64-row sub-tiles (128-byte rows, 128-byte swizzle) and
      // write each with one TMA store (clipped at rows / T).  16x256b TMEM loads give every thread
      // two tokens of two rows (C-fragment layout); stmatrix.trans turns each 8 x 8 block into 8
      // token rows of 8 sign rows (16 bytes), conflict-free under the swizzle.
      const int mi = lane >> 3, mr = lane & 7;  // stmatrix: matrix / memory row this lane addresses
      const uint32_t sub_base = smem_u32(smem) + (uint32_t)(sub >> 1) * (BN * 128);
#pragma unroll
      for (int lb = 0; lb < 2; ++lb) {
        const float rs_lo = __half2float(rs_pre[lb][0]), rs_hi = __half2float(rs_pre[lb][1]);  // rows sub*32 + lb*16 + g (+8)
        const int ch = ((sub & 1) * 32 + lb * 16) / 8 + (mi & 1);  // 16-byte chunk this lane's row lands in
        // all four 32-token loads in flight before one wait (tokens past T are staged too; the
        // TMA store clips them)
        uint32_t v[BN / 64][16];
#pragma unroll
        for (int c = 0; c < BN / 64; ++c)
          tmem_ld16x256_x4(tmem + ((uint32_t)(sub * 32 + lb * 16) << 16) + kAccCol + mh * BN + half * (BN / 2) + c * 32,
                           v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) {
          const int col = half * (BN / 2) + c * 32;
#pragma unroll
          for (int gp = 0; gp < 2; ++gp) {  // 16 tokens per stmatrix.x4
            uint32_t m[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // matrix q: token group 2gp + q/2, rows lo (q even) / hi
              const uint32_t* f = v[c] + 4 * (2 * gp + (q >> 1)) + 2 * (q & 1);
              const float rs = (q & 1) ? rs_hi : rs_lo;
              const __half2 h = __floats2half2_rn(__uint_as_float(f[0]) * rs, __uint_as_float(f[1]) * rs);
              m[q] = *reinterpret_cast<const uint32_t*>(&h);
            }
            const int tk = col + 16 * gp + 8 * (mi >> 1) + mr;
            stmatrix_x4_trans(sub_base + (uint32_t)tk * 128 + (uint32_t)((ch ^ (tk & 7)) * 16), m[0], m[1], m[2], m[3]);
          }
        }
      }
      fence_proxy_async_smem();
      if (threadIdx.x == 32 * kExpWarp0) CT(10);
      asm volatile("bar.sync 1, %0;" ::"n"(kExpWarps * 32) : "memory");
      if (threadIdx.x == 32 * kExpWarp0) {
        CT(11);
        tma_store_2d(&out_map, smem, row0, tok0);
        if (row0 + 64 < p.rows) tma_store_2d(&out_map, smem + BN * 128, row0 + 64, tok0);
        bulk_commit_group();
        bulk_wait_group_read0();
        CT(12);
      }
    }
    float* part = p.part ? p.part + (size_t)blockIdx.z * p.T * p.rows : nullptr;
#pragma unroll 1
    for (int c = 0; c < (p.tma_out ? 0 : BN / 64); ++c) {
      const int col = half * (BN / 2) + c * 32;
      if (tok0 + col >= p.T) break;  // columns past the tokens present (the MMA N may be smaller)
      uint32_t acc[32];
      tmem_ld32(tmem + lane_addr + kAccCol + mh * BN + col, acc);
      tmem_wait_ld();
      if (live) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int tok = tok0 + col + j;
          if (tok < p.T) {
            if (part) part[(size_t)tok * p.rows + grow] = __uint_as_float(acc[j]);
            else p.out[(int64_t)tok * p.ldo + grow] = __float2half_rn(__uint_as_float(acc[j]) * rs);
          }
        }
      }
    }
    if (threadIdx.x == 32 * kExpWarp0) CT(9);
  }
  tc_fence_before();
  __syncthreads();
#ifdef DBF_PREFILL_TRACE
  if (threadIdx.x == 0 && p.trace) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta < 4096) {
      unsigned long long t1, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      asm volatile("{.reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r;}" : "=l"(smid));
      long long* c = cslot;
      c[0] = (long long)cta_t0, c[1] = (long long)t1, c[2] = clock64(), c[3] = (long long)smid;
    }
  }
#endif
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
static int make_act_map(CUtensorMap* map, const void* act, int64_t T, int64_t K, int64_t ld, int box_rows = BN) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return DBF_ERR_CUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(act), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? DBF_OK : DBF_ERR_CUDA;
}

// out: T x rows fp16, row stride ldo elements; box = 64 rows x BN tokens (half a tile), 128-byte swizzle
static int make_out_map(CUtensorMap* map, void* out, int64_t T, int64_t rows, int64_t ldo, int box_tokens = BN) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return DBF_ERR_CUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)ldo * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_tokens};  // 64 rows = one 128-byte swizzle span
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? DBF_OK : DBF_ERR_CUDA;
}

static long long* trace_buf = nullptr;

// out[tok][row] = fp16(rscale[row] * sum_z part[z][tok][row]), splits summed in order (deterministic)
__global__ void split_reduce_kernel(const float* __restrict__ part, int splits, int T, int rows,
                                    const __half* __restrict__ rscale, __half* __restrict__ out, int64_t ldo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)T * rows) return;
  const int row = (int)(i % rows);
  const int64_t tok = i / rows;
  float v = 0.f;
  for (int z = 0; z < splits; ++z) v += __ldcs(part + (size_t)z * T * rows + i);
  out[tok * ldo + row] = __float2half_rn(v * (rscale ? __half2float(rscale[row]) : 1.f));
}

// K splits for a launch of `tiles` output tiles: enough CTAs to cover the SMs once, each split a
// whole number of K-block pairs and at least kMinSplitKb K blocks.  1 = no split.
constexpr int kMinSplitKb = 8;
inline int split_count(int64_t tiles, int num_kb, int* kb_per_split) {
  int S = (int)std::max<int64_t>(1, kNumSMs / std::max<int64_t>(tiles, 1));
  S = std::min(S, std::max(1, num_kb / kMinSplitKb));
  int kps = (int)ceil_div(num_kb, S);
  kps += kps & 1;
  S = (int)ceil_div(num_kb, kps);
  *kb_per_split = kps;
  return S;
}
inline size_t split_bytes(int64_t T, int64_t K, int64_t rows) {
  if (T > BN) return 0;  // large token counts fill the GPU with token tiles
  int kps = 0;
  const int S = split_count(ceil_div(rows, BM), (int)ceil_div(K, BK), &kps);
  return S > 1 ? (size_t)S * T * rows * sizeof(float) : 0;
}

static int launch_sign_gemm(const void* act, int64_t T, int64_t K, int64_t ld_act, const uint32_t* words,
                            int64_t pitch, int64_t rows, const __half* kscale, const __half* rscale, __half* out,
                            int64_t ldo, cudaStream_t stream, float* split_ws = nullptr, size_t split_ws_bytes = 0) {
  if (T < 1 || K < 1 || rows < 1) return DBF_ERR_INVALID_ARGUMENT;
  if ((ld_act * 2) % 16 != 0 || ((uintptr_t)act & 15) != 0 || ld_act < K) return DBF_ERR_UNSUPPORTED;
  if (((uintptr_t)words & 15) != 0 || pitch % 4 != 0) return DBF_ERR_UNSUPPORTED;
  if (pitch * 32 < ceil_div(K, BK) * BK) return DBF_ERR_SHAPE;  // a K block would read past the row
  if (T > INT32_MAX || rows > INT32_MAX || K > INT32_MAX) return DBF_ERR_UNSUPPORTED;
  // T <= BN: one token tile whose MMA N / activation box cover only the tokens present
  const bool small = T <= kSmallBN;
  const int n_mma = T >= BN ? BN : (int)ceil_div(T, 16) * 16;
  CUtensorMap map;
  int st = make_act_map(&map, act, T, K, ld_act, n_mma);
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
  p.n_mma = n_mma;
  p.act_bytes = n_mma * BK * 2;
  p.kb_per_split = p.num_kb;
  p.part = nullptr;
  int splits = 1;
  if (T <= BN) {
    int kps = 0;
    const int S = split_count(ceil_div(rows, BM), p.num_kb, &kps);
    if (S > 1 && split_ws && split_ws_bytes >= (size_t)S * T * rows * sizeof(float)) {
      splits = S;
      p.kb_per_split = kps;
      p.part = split_ws;
    }
  }
  // TMA-store epilogue: full-size tiles writing fp16 with a 16-byte row stride (the staged tile,
  // BN x BM fp16 = 64 KB, lives in the activation ring)
  CUtensorMap omap;
  std::memset(&omap, 0, sizeof(omap));
  p.tma_out = 0;
  if (!small && splits == 1 && (ldo * 2) % 16 == 0 && ((uintptr_t)out & 15) == 0 &&
      (size_t)STAGES * BN * BK * 2 >= (size_t)BM * BN * 2) {
    st = make_out_map(&omap, out, T, rows, ldo);
    if (st != DBF_OK) return st;
    p.tma_out = 1;
  }
  p.trace = nullptr;
#ifdef DBF_PREFILL_TRACE  // diagnostics build only (tools/prefill_trace.py)
  {
    if (!trace_buf) cudaMalloc(&trace_buf, 8 * 24 * 4096);
    p.trace = trace_buf;
  }
#endif
  const unsigned gx = (unsigned)ceil_div(rows, BM);
  dim3 grid(gx, (unsigned)ceil_div(T, small ? kSmallBN : BN), (unsigned)splits);
  const bool ks_smem = false;  // K scales are register-resident (shuffled), no shared-memory copy
  // the small configuration pads its shared memory so that one CTA per SM owns all of TMEM
  const size_t smem = small ? std::max<size_t>(smem_bytes_for<kSmallBN, kSmallStages>(p.num_kb, ks_smem), 120 * 1024)
                            : smem_bytes(p.num_kb, ks_smem);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, map, omap, p);
  };
  cudaError_t e;
  if (small)
    e = kscale ? go(sign_gemm_kernel<true, kSmallBN, kSmallStages>)
               : go(sign_gemm_kernel<false, kSmallBN, kSmallStages>);
  else e = kscale ? go(sign_gemm_kernel<true>) : go(sign_gemm_kernel<false>);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  st = check_launch();
  if (st != DBF_OK || splits == 1) return st;
  const int64_t total = T * rows;
  split_reduce_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, stream>>>(p.part, splits, (int)T, (int)rows, rscale,
                                                                          out, ldo);
  return check_launch();
}

// ================================================================================================
// The whole layer in ONE persistent launch (T > 256 tokens):
//
//   GEMM1 tiles 0 .. N1-1        t[T, k] = mid (.) (X . (B (.) b)^T)    token-block-major order
//   GEMM2 tiles N1 .. N1+N2-1    Y[T, n] = a (.) (t . A^T)
//
// claimed dynamically by one CTA per SM (a global tile counter).  Traced on the per-tile kernel
// (tools/prefill_ctas.py): a 128 x 256 tile spends 2.7 us before its first MMA and 2.4 us after its
// last one, and 128-192 tiles on 148 SMs leave whole waves idle, so a 7B q layer took 67 us for 40
// us of MMA K loops.  Here a GEMM2 tile of token block tb only waits for the k/128 GEMM1 tiles of
// tb (per-token-block counters, release/acquire), the epilogue has its own 4 warps that drain the
// accumulator into registers (the MMA's only wait) and store straight to global memory while the
// next tile's K loop runs, and the activation ring and the sign expansion run continuously across
// tiles.  Tile mechanics and numerics are the per-tile kernel's (same K order, fp32 TMEM
// accumulation, same rounding): the outputs are bitwise those of the two-launch path.
//
// Warp roles (16 warps): lanes of warps 0, 2, 3 issue the activation TMA loads (one issuer per ring
// stage -- a thread's TMA loads complete one after another; issuer 0 also claims the tiles),
// warp 1 allocates TMEM and issues the MMAs, 4..11 expand signs, 12..15 run the epilogue.
namespace layer {

constexpr int S = 6;                            // ring stages (32 KB activation box + 32-column TMEM A slot)
constexpr int kStagingBytes = 128 * 128 * 2;    // half a tile: fp16 [128 tokens][128 rows], two 64-row TMA boxes
constexpr int kActBytes = 256 * BK * 2;         // one 256-token x 64-column fp16 box
constexpr int kACol0 = 256;                     // A slots after the 256-column accumulator
constexpr int kExp0 = 4, kExpN = 8, kEpi0 = 12, kEpiN = 4;
constexpr int kThreadsL = 16 * 32;
constexpr int kRing = 2;                        // tile-id ring
constexpr int kIssuers = S;                     // lanes 0-1 of warps 0, 2, 3
static_assert(kIssuers <= 6, "issuers are lanes 0-1 of warps 0, 2 and 3");
static_assert(kACol0 + S * kAColsPerHalf <= kTmemCols, "TMEM budget");

struct LParams {
  const uint32_t* B_words; int64_t B_pitch;     // k x m paired words
  const uint32_t* A_words; int64_t A_pitch;     // n x k paired words
  const __half* a; const __half* mid; const __half* b;
  __half* t; int64_t ldt;                       // GEMM1 output (GEMM2 input, read back through t_map)
  __half* Y; int64_t ldy;
  int n, k, m, T;
  int rt1, rt2, tbs;                            // row tiles of GEMM1 (k/128), GEMM2 (n/128); token blocks
  int nkb1, nkb2;                               // K blocks of GEMM1 (m/64) and GEMM2 (k/64)
  int* sched;                                   // [0] tile counter, [1..tbs] GEMM1 tiles done per token block
  long long* trace;                             // debug: per-tile globaltimer stamps, or nullptr
  long long* ktrace;                            // debug: per-K-block clock64 stamps of CTA 0 (first 1024), or nullptr
};

struct __align__(8) LBar {
  uint64_t full_act[S], full_a[S], empty[S];
  uint64_t acc_full, acc_empty;
  uint64_t tile_full[kRing], tile_empty[kRing];
  int tile_id[kRing];
  uint32_t tmem_base;
};

inline size_t layer_smem_bytes() { return 1024 + (size_t)S * kActBytes + kStagingBytes + sizeof(LBar); }

struct Tile {
  int g1;      // 1: GEMM1, 0: GEMM2
  int rt, tb;
  bool valid;
};
__device__ __forceinline__ Tile decode(const LParams& p, int t) {
  Tile ti;
  const int n1 = p.rt1 * p.tbs;
  ti.valid = t >= 0 && t < n1 + p.rt2 * p.tbs;
  if (t < n1) {
    ti.g1 = 1, ti.tb = t / p.rt1, ti.rt = t % p.rt1;
  } else {
    t -= n1;
    ti.g1 = 0, ti.tb = t / p.rt2, ti.rt = t % p.rt2;
  }
  return ti;
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// the tile id of local tile j (whole warp; lane 0 waits), then this warp is done reading the slot
__device__ __forceinline__ int warp_read_tile(LBar& bar, int j, int lane) {
  const int slot = j % kRing;
  if (lane == 0) mbar_wait(&bar.tile_full[slot], (j / kRing) & 1);
  __syncwarp();
  const int t = *reinterpret_cast<volatile int*>(&bar.tile_id[slot]);
  __syncwarp();
  if (lane == 0) mbar_arrive(&bar.tile_empty[slot]);
  return t;
}

__global__ void __launch_bounds__(kThreadsL, 1)
    sign_layer_kernel(const __grid_constant__ CUtensorMap x_map, const __grid_constant__ CUtensorMap t_map,
                      const __grid_constant__ CUtensorMap t_store, const __grid_constant__ CUtensorMap y_store,
                      const LParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* act = smem;
  uint8_t* staging = smem + (size_t)S * kActBytes;
  LBar& bar = *reinterpret_cast<LBar*>(staging + kStagingBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&bar.full_act[s], 1);
      mbar_init(&bar.full_a[s], kExpN);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc_full, 1);
    mbar_init(&bar.acc_empty, kEpiN);
    for (int j = 0; j < kRing; ++j) {
      mbar_init(&bar.tile_full[j], 1);
      // the other issuers + MMA thread + expander warps + epilogue warps
      mbar_init(&bar.tile_empty[j], (kIssuers - 1) + 1 + kExpN + kEpiN);
    }
    fence_mbar_init();
    tma_prefetch_desc(&x_map);
    tma_prefetch_desc(&t_map);
    tma_prefetch_desc(&t_store);
    tma_prefetch_desc(&y_store);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp == 0 || warp == 2 || warp == 3) {
    // ---------------- TMA issuers (issuer 0 also schedules) ----------------
    const int issuer = (warp == 0 ? 0 : warp - 1) * 2 + lane;
    if (lane < 2 && issuer < kIssuers) {
      const uint64_t pol = policy_evict_last();  // activations are re-read by every row tile
      asm volatile("griddepcontrol.wait;" ::: "memory");  // the tile counters, X and t belong to the stream
      int g = 0;                                          // ring position (K blocks of all tiles so far)
      for (int j = 0;; ++j) {
        const int slot = j % kRing;
        int t;
        if (issuer == 0) {
          mbar_wait(&bar.tile_empty[slot], ((j / kRing) & 1) ^ 1);
          // claimed once issuer 0 has issued its loads of the current tile (just in time: the ring
          // holds S K blocks, so dynamic claiming balances the tail)
          t = atomicAdd(p.sched, 1);
          bar.tile_id[slot] = t;
          mbar_arrive(&bar.tile_full[slot]);
        } else {
          mbar_wait(&bar.tile_full[slot], (j / kRing) & 1);
          t = *reinterpret_cast<volatile int*>(&bar.tile_id[slot]);
          mbar_arrive(&bar.tile_empty[slot]);
        }
        const Tile ti = decode(p, t);
        if (!ti.valid) break;
        if (issuer == 0 && p.trace) p.trace[8 * t + 0] = gtimer();
        const int nkb = ti.g1 ? p.nkb1 : p.nkb2;
        // this issuer's first K block of the tile: the one landing in ring stage `issuer`
        int kb = ((issuer - g) % S + S) % S;
        if (!ti.g1 && kb < nkb) {  // t of this token block must be complete (the GEMM1 epilogues)
          while (true) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.sched + 1 + ti.tb) : "memory");
            if (v >= p.rt1) break;
            __nanosleep(128);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          if (issuer == 0 && p.trace) p.trace[8 * t + 1] = gtimer();
        }
        const CUtensorMap* map = ti.g1 ? &x_map : &t_map;
        for (; kb < nkb; kb += S) {
          const int gg = g + kb;
          const int s = gg % S;
          const uint32_t ph = (gg / S) & 1;
          mbar_wait(&bar.empty[s], ph ^ 1);
          if (p.ktrace && blockIdx.x == 0 && gg < 1024) p.ktrace[4 * gg + 0] = clock64();
          mbar_arrive_expect_tx(&bar.full_act[s], kActBytes);
          tma_load_2d(act + (size_t)s * kActBytes, map, kb * BK, ti.tb * 256, &bar.full_act[s], pol);
        }
        g += nkb;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(UM, 256);
      int g = 0;
      for (int j = 0;; ++j) {
        const int slot = j % kRing;
        mbar_wait(&bar.tile_full[slot], (j / kRing) & 1);
        const int t = *reinterpret_cast<volatile int*>(&bar.tile_id[slot]);
        mbar_arrive(&bar.tile_empty[slot]);
        const Tile ti = decode(p, t);
        if (!ti.valid) break;
        const int nkb = ti.g1 ? p.nkb1 : p.nkb2;
        mbar_wait(&bar.acc_empty, (j & 1) ^ 1);  // the epilogue drained the previous tile's accumulator
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          const uint32_t ph = (g / S) & 1;
          mbar_wait(&bar.full_act[s], ph);
          if (p.ktrace && blockIdx.x == 0 && g < 1024) p.ktrace[4 * g + 1] = clock64();
          mbar_wait(&bar.full_a[s], ph);
          if (p.ktrace && blockIdx.x == 0 && g < 1024) p.ktrace[4 * g + 2] = clock64();
          tc_fence_after();
          if (kb == 0 && p.trace) p.trace[8 * t + 2] = gtimer();
          const uint32_t a_base = tmem + kACol0 + s * kAColsPerHalf;
          const uint32_t b_base = smem_u32(act + (size_t)s * kActBytes);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk)
            mma_f16_ts(tmem, a_base + kk * (UK / 2), sdesc_k_sw128(b_base + kk * UK * 2), idesc, (kb | kk) != 0);
          mma_commit(&bar.empty[s]);
        }
        mma_commit(&bar.acc_full);
        if (p.trace) p.trace[8 * t + 3] = gtimer();
      }
    }
  } else if (warp >= kExp0 && warp < kExp0 + kExpN) {
    // ---------------- sign expanders (the per-tile kernel's loop, ring position carried across tiles) ----
    const int sub = warp & 3, half = (warp - kExp0) >> 2;
    const uint32_t col = tmem + ((uint32_t)(sub * 32) << 16) + kACol0 + half * 16;
    int g = 0;
    for (int j = 0;; ++j) {
      const int t = warp_read_tile(bar, j, lane);
      const Tile ti = decode(p, t);
      if (!ti.valid) break;
      const int rows = ti.g1 ? p.k : p.n, nkb = ti.g1 ? p.nkb1 : p.nkb2;
      const int grow = ti.rt * UM + sub * 32 + lane;
      const bool live = grow < rows;
      const uint4* wrow = reinterpret_cast<const uint4*>((ti.g1 ? p.B_words : p.A_words) +
                                                         (int64_t)(live ? grow : 0) * (ti.g1 ? p.B_pitch : p.A_pitch));
      const bool has_ks = ti.g1 && p.b != nullptr;  // GEMM1's K scale b; GEMM2 has none
      const int nquads = (nkb + 1) >> 1;
      // K scales live in registers: for the 8 K blocks of a group, lane L holds in ksr[jp] the fp16 pair
      // (L & 15) of this warp's 32 columns of K block kg + 2 jp + (L >> 4); a K block's 16 pairs are
      // then one shuffle each (no shared memory for them, no L1 traffic in the loop)
      const unsigned short* bsrc = reinterpret_cast<const unsigned short*>(p.b);
      auto load_ksr = [&](int kg, uint32_t (&r)[4]) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const int c = (kg + 2 * jp + (lane >> 4)) * BK + half * 32 + 2 * (lane & 15);
          r[jp] = !has_ks ? 0x3C003C00u
                          : ((c < p.m ? (uint32_t)__ldg(bsrc + c) : 0u) |
                             ((c + 1 < p.m ? (uint32_t)__ldg(bsrc + c + 1) : 0u) << 16));
        }
      };
      uint32_t ksr[4];
      load_ksr(0, ksr);
      uint4 q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = (live && i < nquads) ? __ldg(wrow + i) : make_uint4(0, 0, 0, 0);
      for (int kg = 0; kg < nkb; kg += 8) {
        uint4 nq[4];
        uint32_t nksr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int qi = (kg >> 1) + 4 + i;
          nq[i] = (live && qi < nquads) ? __ldg(wrow + qi) : make_uint4(0, 0, 0, 0);
        }
        load_ksr(kg + 8, nksr);
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const int kb = kg + 2 * jp;
          if (kb >= nkb) break;
          const bool two = kb + 1 < nkb;
          const int s0 = g % S, s1 = (g + 1) % S;
          const uint32_t ph0 = (g / S) & 1, ph1 = ((g + 1) / S) & 1;
          uint32_t ks[16], v0[16], v1[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) ks[w] = __shfl_sync(0xffffffffu, ksr[jp], w);
          expand_word(half ? q[jp].y : q[jp].x, ks, v0);
          if (two) {
#pragma unroll
            for (int w = 0; w < 16; ++w) ks[w] = __shfl_sync(0xffffffffu, ksr[jp], 16 + w);
            expand_word(half ? q[jp].w : q[jp].z, ks, v1);
          }
          if (lane == 0) {
            mbar_wait(&bar.empty[s0], ph0 ^ 1);
            if (two) mbar_wait(&bar.empty[s1], ph1 ^ 1);
          }
          __syncwarp();
          tc_fence_after();
          tmem_st16(col + s0 * kAColsPerHalf, v0);
          if (two) tmem_st16(col + s1 * kAColsPerHalf, v1);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&bar.full_a[s0]);
            if (two) mbar_arrive(&bar.full_a[s1]);
            if (p.ktrace && blockIdx.x == 0 && warp == kExp0 && g < 1023) p.ktrace[4 * g + 3] = p.ktrace[4 * g + 7] = clock64();
          }
          g += two ? 2 : 1;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = nq[i], ksr[i] = nksr[i];
      }
    }
  } else if (warp >= kEpi0) {
    // ---------------- epilogue: accumulator -> fp16 staging (half a tile) -> TMA stores ----------------
    // 16x256b TMEM loads give every thread two tokens of two rows (C-fragment layout); stmatrix.trans
    // turns each 8 x 8 block into 8 token rows of 8 sign rows in the staging tile ([token][row],
    // 128-byte rows, 128-byte swizzle: two 64-row TMA boxes of 128 tokens).  Tokens 0-127 go through
    // staging first; tokens 128-255 are converted to fp16 in registers, the accumulator is released
    // (the next tile's MMAs start), and they are staged once the first stores have read the tile.
    const int sub = warp & 3;
    const bool storer = threadIdx.x == kEpi0 * 32;
    const int mi = lane >> 3, mr = lane & 7;  // stmatrix: matrix / memory row this lane addresses
    const uint32_t sub_base = smem_u32(staging) + (uint32_t)(sub >> 1) * (128 * 128);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel may still read t / Y
    for (int j = 0;; ++j) {
      const int t = warp_read_tile(bar, j, lane);
      const Tile ti = decode(p, t);
      if (!ti.valid) break;
      const int rows = ti.g1 ? p.k : p.n;
      const __half* rsrc = ti.g1 ? p.mid : p.a;
      const CUtensorMap* om = ti.g1 ? &t_store : &y_store;
      float rs[2][2];
#pragma unroll
      for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
          const int rr = ti.rt * UM + sub * 32 + lb * 16 + hi * 8 + (lane >> 2);
          rs[lb][hi] = rr < rows ? __half2float(rsrc[rr]) : 0.f;
        }
      // stmatrix of one 32-token group (16 packed registers: gp x qd) of row group lb at token tk0
      auto stage = [&](int lb, int tk0, const uint32_t (&mm)[8]) {
        const int ch = ((sub & 1) * 32 + lb * 16) / 8 + (mi & 1);
#pragma unroll
        for (int gp = 0; gp < 2; ++gp) {
          const int tk = tk0 + 16 * gp + 8 * (mi >> 1) + mr;
          stmatrix_x4_trans(sub_base + (uint32_t)tk * 128 + (uint32_t)((ch ^ (tk & 7)) * 16), mm[4 * gp], mm[4 * gp + 1],
                            mm[4 * gp + 2], mm[4 * gp + 3]);
        }
      };
      auto pack = [&](int lb, const uint32_t (&v)[16], uint32_t (&mm)[8]) {
#pragma unroll
        for (int gp = 0; gp < 2; ++gp)
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {  // matrix qd: token group 2gp + qd/2, rows lo (qd even) / hi
            const uint32_t* f = v + 4 * (2 * gp + (qd >> 1)) + 2 * (qd & 1);
            const float r = rs[lb][qd & 1];
            const __half2 h = __floats2half2_rn(__uint_as_float(f[0]) * r, __uint_as_float(f[1]) * r);
            mm[4 * gp + qd] = *reinterpret_cast<const uint32_t*>(&h);
          }
      };
      if (storer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free again
      if (lane == 0) {  // a long wait (a whole K loop): back off instead of spinning next to the MMA issuer
        while (!mbar_test(&bar.acc_full, j & 1)) __nanosleep(256);
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiN * 32) : "memory");
      tc_fence_after();
      if (storer && p.trace) p.trace[8 * t + 4] = gtimer();
      // phase A: tokens 0-127 straight into staging
#pragma unroll
      for (int lb = 0; lb < 2; ++lb) {
        uint32_t v[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld16x256_x4(tmem + ((uint32_t)(sub * 32 + lb * 16) << 16) + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t mm[8];
          pack(lb, v[c], mm);
          stage(lb, c * 32, mm);
        }
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiN * 32) : "memory");
      if (storer) {
        tma_store_2d(om, staging, ti.rt * UM, ti.tb * 256);
        if (ti.rt * UM + 64 < rows) tma_store_2d(om, staging + 128 * 128, ti.rt * UM + 64, ti.tb * 256);
        bulk_commit_group();
      }
      // phase B: tokens 128-255 into registers as fp16, then the accumulator is free
      uint32_t hold[2][4][8];
#pragma unroll
      for (int lb = 0; lb < 2; ++lb) {
        uint32_t v[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld16x256_x4(tmem + ((uint32_t)(sub * 32 + lb * 16) << 16) + 128 + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) pack(lb, v[c], hold[lb][c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.acc_empty);
      if (storer && p.trace) p.trace[8 * t + 6] = gtimer();
      if (storer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // phase A's stores read the tile
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiN * 32) : "memory");
#pragma unroll
      for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int c = 0; c < 4; ++c) stage(lb, c * 32, hold[lb][c]);
      fence_proxy_async_smem();
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiN * 32) : "memory");
      if (storer) {
        tma_store_2d(om, staging, ti.rt * UM, ti.tb * 256 + 128);
        if (ti.rt * UM + 64 < rows) tma_store_2d(om, staging + 128 * 128, ti.rt * UM + 64, ti.tb * 256 + 128);
        bulk_commit_group();
        if (ti.g1) {  // publish t of this tile before counting it done
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.sched + 1 + ti.tb) : "memory");
        }
        if (p.trace) p.trace[8 * t + 5] = gtimer();
      }
    }
    if (storer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

inline size_t counter_bytes(int64_t tokens) { return (size_t)(ceil_div(tokens, 256) + 1) * 4; }

#ifdef DBF_PREFILL_TRACE
static long long* layer_trace = nullptr;
#endif

// Both GEMMs of one layer as one persistent launch.  t: T x ldt fp16 workspace, counters: zeroed here.
static int launch_layer(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired, int64_t B_pitch,
                        const __half* a, const __half* mid, const __half* b, int64_t n, int64_t k, int64_t m,
                        const void* X, int64_t T, int64_t ldx, void* Y, int64_t ldy, __half* t, int64_t ldt,
                        int* counters, cudaStream_t stream) {
  CUtensorMap xm, tm, ts, ys;
  int st = make_act_map(&xm, X, T, m, ldx, 256);
  if (st == DBF_OK) st = make_act_map(&tm, t, T, k, ldt, 256);
  if (st == DBF_OK) st = make_out_map(&ts, t, T, k, ldt, 128);
  if (st == DBF_OK) st = make_out_map(&ys, Y, T, n, ldy, 128);
  if (st != DBF_OK) return st;
  LParams p;
  p.B_words = B_paired, p.B_pitch = B_pitch, p.A_words = A_paired, p.A_pitch = A_pitch;
  p.a = a, p.mid = mid, p.b = b;
  p.t = t, p.ldt = ldt, p.Y = (__half*)Y, p.ldy = ldy;
  p.n = (int)n, p.k = (int)k, p.m = (int)m, p.T = (int)T;
  p.rt1 = (int)ceil_div(k, UM), p.rt2 = (int)ceil_div(n, UM), p.tbs = (int)ceil_div(T, 256);
  p.nkb1 = (int)ceil_div(m, BK), p.nkb2 = (int)ceil_div(k, BK);
  p.sched = counters;
  p.trace = nullptr;
  p.ktrace = nullptr;
#ifdef DBF_PREFILL_TRACE
  {
    const size_t need = 8 * sizeof(long long) * (size_t)(p.rt1 + p.rt2) * p.tbs + 4 * 1024 * 8;
    static size_t have = 0;
    if (need > have) {
      if (layer_trace) cudaFree(layer_trace);
      cudaMalloc(&layer_trace, need);
      have = need;
    }
    p.trace = layer_trace;
    p.ktrace = layer_trace + 8 * (size_t)(p.rt1 + p.rt2) * p.tbs;
  }
#endif
  cudaError_t e = cudaMemsetAsync(counters, 0, counter_bytes(T), stream);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (int64_t)(p.rt1 + p.rt2) * p.tbs;
  const size_t smem = layer_smem_bytes();
  e = cudaFuncSetAttribute(sign_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>(tiles, sms));
  cfg.blockDim = dim3(kThreadsL);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, sign_layer_kernel, xm, tm, ts, ys, p);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  return check_launch();
}

}  // namespace layer

}  // namespace prefill
}  // namespace dbf

using namespace dbf;

extern "C" {

// debug: copy the last traced launch's stamps (5 * num_kb int64) to host memory
int dbf_prefill_debug_trace(long long* host, int n) {
  if (!prefill::trace_buf) return DBF_ERR_UNSUPPORTED;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, prefill::trace_buf, 8 * (size_t)n, cudaMemcpyDeviceToHost) == cudaSuccess ? DBF_OK
                                                                                                    : DBF_ERR_CUDA;
}

#ifdef DBF_PREFILL_TRACE
// debug: per-tile {claim, dependency met, first MMA, last commit, accumulator seen, stored} globaltimer
// stamps of the last one-launch layer (8 int64 per tile)
int dbf_prefill_debug_layer(long long* host, int n) {
  if (!prefill::layer::layer_trace) return DBF_ERR_UNSUPPORTED;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, prefill::layer::layer_trace, 8 * (size_t)n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? DBF_OK : DBF_ERR_CUDA;
}
// debug: per-CTA {globaltimer start, end, clock end, smid, clock start, setup done, first MMA, last commit,
// accumulator seen, -} of the last traced launch
int dbf_prefill_debug_ctas(long long* host, int n) {
  if (!prefill::trace_buf) return DBF_ERR_UNSUPPORTED;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, prefill::trace_buf + 6 * 4096, 8 * (size_t)n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? DBF_OK : DBF_ERR_CUDA;
}
#endif

int64_t dbf_prefill_ld(int64_t cols) { return ceil_div(cols, 64) * 64; }

size_t dbf_prefill_workspace_bytes(int64_t k, int64_t tokens) {
  return (size_t)(tokens > 0 ? tokens : 0) * (size_t)dbf_prefill_ld(k) * 2;
}

int dbf_sign_gemm(const void* act, int64_t tokens, int64_t K, int64_t ld_act, const uint32_t* paired,
                  int64_t word_pitch, int64_t rows, const void* kscale, const void* rscale, void* out, int64_t ldo,
                  void* stream) {
  if (!act || !paired || !out) return DBF_ERR_INVALID_ARGUMENT;
  if (ldo < rows) return DBF_ERR_SHAPE;
  return prefill::launch_sign_gemm(act, tokens, K, ld_act, paired, word_pitch, rows, (const __half*)kscale,
                                   (const __half*)rscale, (__half*)out, ldo, (cudaStream_t)stream);
}

size_t dbf_prefill_workspace_bytes_nkm(int64_t n, int64_t k, int64_t m, int64_t tokens) {
  if (n < 1 || k < 1 || m < 1 || tokens < 1) return 0;
  const size_t t = (dbf_prefill_workspace_bytes(k, tokens) + 255) & ~(size_t)255;
  // T <= 256: split-K partials; above: the one-launch layer kernel's tile counters
  return t + std::max({prefill::split_bytes(tokens, m, k), prefill::split_bytes(tokens, k, n),
                       tokens > prefill::BN ? prefill::layer::counter_bytes(tokens) : (size_t)0});
}

int dbf_prefill_layer_path(int64_t n, int64_t k, int64_t m, int64_t tokens) {
  if (n < 1 || k < 1 || m < 1 || tokens <= prefill::BN) return DBF_PREFILL_TWO_LAUNCHES;
  // Measured on the Llama-2-7B shapes at T = 2048 (tools/prefill_ab.py): the one-launch
  // kernel wins where GEMM1's tiles spill into a second, partly idle wave (gate/up 1235 vs 1130 TF/s,
  // down 1063 vs 1057) and loses where GEMM1 fits one wave (q 929 vs 1061: the CTAs beyond GEMM1's
  // tiles wait for t, and its K loop runs ~10 % slower than the per-tile kernel's).
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles1 = ceil_div(k, prefill::UM) * ceil_div(tokens, prefill::BN);
  return tiles1 > sms ? DBF_PREFILL_ONE_LAUNCH : DBF_PREFILL_TWO_LAUNCHES;
}

int dbf_forward_prefill(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired, int64_t B_pitch,
                        const void* a, const void* mid, const void* b, int64_t n, int64_t k, int64_t m,
                        const void* X, int64_t tokens, int64_t ldx, void* Y, int64_t ldy, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return dbf_forward_prefill_ex(A_paired, A_pitch, B_paired, B_pitch, a, mid, b, n, k, m, X, tokens, ldx, Y, ldy,
                                workspace, workspace_bytes, DBF_PREFILL_AUTO, stream);
}

int dbf_forward_prefill_ex(const uint32_t* A_paired, int64_t A_pitch, const uint32_t* B_paired, int64_t B_pitch,
                           const void* a, const void* mid, const void* b, int64_t n, int64_t k, int64_t m,
                           const void* X, int64_t tokens, int64_t ldx, void* Y, int64_t ldy, void* workspace,
                           size_t workspace_bytes, int path, void* stream) {
  if (path != DBF_PREFILL_AUTO && path != DBF_PREFILL_TWO_LAUNCHES && path != DBF_PREFILL_ONE_LAUNCH)
    return DBF_ERR_INVALID_ARGUMENT;
  if (!A_paired || !B_paired || !a || !mid || !b || !X || !Y) return DBF_ERR_INVALID_ARGUMENT;
  if (n < 1 || k < 1 || m < 1 || tokens < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (ldy < n || ldx < m) return DBF_ERR_SHAPE;
  if (A_pitch < canonical_pitch(k) || B_pitch < canonical_pitch(m)) return DBF_ERR_SHAPE;
  if (!workspace || workspace_bytes < dbf_prefill_workspace_bytes(k, tokens)) return DBF_ERR_WORKSPACE;
  const int64_t ldt = dbf_prefill_ld(k);
  __half* t = (__half*)workspace;
  cudaStream_t s = (cudaStream_t)stream;
  // split-K partials after t when the workspace has room (dbf_prefill_workspace_bytes_nkm)
  const size_t tb = (dbf_prefill_workspace_bytes(k, tokens) + 255) & ~(size_t)255;
  float* sw = workspace_bytes > tb ? (float*)((char*)workspace + tb) : nullptr;
  const size_t swb = workspace_bytes > tb ? workspace_bytes - tb : 0;
  // more than one token tile: both GEMMs in one persistent launch when the workspace holds its tile
  // counters and t / Y suit the TMA stores (16-byte aligned rows)
  if (path == DBF_PREFILL_AUTO) path = dbf_prefill_layer_path(n, k, m, tokens);
  const bool layer_ok =
      tokens > prefill::BN && swb >= prefill::layer::counter_bytes(tokens) && (ldy * 2) % 16 == 0 &&
      ((uintptr_t)Y & 15) == 0 && (ldx * 2) % 16 == 0 && ((uintptr_t)X & 15) == 0 &&
      A_pitch * 32 >= ceil_div(k, prefill::BK) * prefill::BK && B_pitch * 32 >= ceil_div(m, prefill::BK) * prefill::BK &&
      ((uintptr_t)A_paired & 15) == 0 && ((uintptr_t)B_paired & 15) == 0 && A_pitch % 4 == 0 && B_pitch % 4 == 0 &&
      tokens <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX && m <= INT32_MAX;
  if (path == DBF_PREFILL_ONE_LAUNCH && !layer_ok) return DBF_ERR_UNSUPPORTED;
  if (path == DBF_PREFILL_ONE_LAUNCH)
    return prefill::layer::launch_layer(A_paired, A_pitch, B_paired, B_pitch, (const __half*)a, (const __half*)mid,
                                        (const __half*)b, n, k, m, X, tokens, ldx, Y, ldy, t, ldt, (int*)sw, s);
  int st = prefill::launch_sign_gemm(X, tokens, m, ldx, B_paired, B_pitch, k, (const __half*)b,
                                     (const __half*)mid, t, ldt, s, sw, swb);
  if (st != DBF_OK) return st;
  return prefill::launch_sign_gemm(t, tokens, k, ldt, A_paired, A_pitch, n, nullptr, (const __half*)a,
                                   (__half*)Y, ldy, s, sw, swb);
}

}  // extern "C"
