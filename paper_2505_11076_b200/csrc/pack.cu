// Sign packing kernels: the B200 replacement of bitcore.pack / bitcore.unpack
// (/root/reference/pkg/src/dbf/bitcore.py:72-91) plus the conversions between the reference's
// uint8 row bytes, the canonical uint32 device layout and the tiled decode layout.
#include <algorithm>
#include "common.cuh"

namespace dbf {

// ---- pack: one warp per 256-column segment of a row.  Lane l loads the 8 values of columns
// 8l..8l+7 (one 16-byte load for fp16/bf16, two for fp32, four for fp64 when the row is aligned),
// tests them on their raw bits (|v| == 1 exactly: NaN and 0 rejected, bitcore.py:79-80) and
// builds byte l of the segment; four lanes' bytes are one 32-bit word (bit i <-> column
// 32 * word + i, LSB-first, bitcore.py:7-9).  The first offending row-major index goes to
// *first_bad by a 64-bit atomicMin.
template <typename T> struct SignBits;
template <> struct SignBits<__half> { using U = uint16_t; static constexpr U kAbs = 0x7FFF, kOne = 0x3C00, kSign = 0x8000; };
template <> struct SignBits<__nv_bfloat16> { using U = uint16_t; static constexpr U kAbs = 0x7FFF, kOne = 0x3F80, kSign = 0x8000; };
template <> struct SignBits<float> { using U = uint32_t; static constexpr U kAbs = 0x7FFFFFFFu, kOne = 0x3F800000u, kSign = 0x80000000u; };
template <> struct SignBits<double> {
  using U = unsigned long long;
  static constexpr U kAbs = 0x7FFFFFFFFFFFFFFFull, kOne = 0x3FF0000000000000ull, kSign = 0x8000000000000000ull;
};

// Segments per warp per iteration: four 16-byte loads per lane in flight whatever the dtype (fp16 /
// bf16: 4 segments, fp32: 2, fp64: 1); measured against 2 and 8 for fp16 (0.47 / 0.45 vs 0.52 of
// HBM) and against register caps for higher occupancy (6 CTAs/SM 0.37, 8 CTAs/SM 0.35).
template <typename T> constexpr int pack_segs() { return sizeof(T) <= 2 ? 4 : sizeof(T) == 4 ? 2 : 1; }

// I: index type -- int when every element and word offset fits (fewer instructions per segment:
// the loop is issue-bound at fp16), int64_t otherwise
template <typename T, typename I>
__global__ void __launch_bounds__(256) pack_kernel(const T* __restrict__ dense, I rows, I cols, I ld,
                                                   uint32_t* __restrict__ words, I pitch,
                                                   unsigned long long* __restrict__ first_bad, int vec_rows) {
  using SB = SignBits<T>;
  using U = typename SB::U;
  constexpr int SEGS = pack_segs<T>();
  const int lane = threadIdx.x & 31;
  const I spr = (pitch + 7) / 8;  // segments per row: 8 words = 256 columns each
  const I nseg = rows * spr;
  const I nwarps = (I)(((int64_t)gridDim.x * blockDim.x) >> 5);
  // grid-stride over groups of SEGS consecutive segments (mostly of one row: contiguous bytes)
  for (I base = (I)((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * SEGS); base < nseg;
       base += nwarps * SEGS) {
    U v[SEGS][8];
    I rr[SEGS], ss[SEGS];
    {
      I r = base / spr, sg = base - r * spr;
#pragma unroll
      for (int q = 0; q < SEGS; ++q) {  // every load of the group issued before any test
        rr[q] = r, ss[q] = sg;
        if (r < rows) {
          const I c0 = sg * 256 + 8 * lane;
          const U* row = reinterpret_cast<const U*>(dense + r * ld);
          if (vec_rows && c0 + 8 <= cols) {
#pragma unroll
            for (int p = 0; p < (int)(8 * sizeof(U) / 16); ++p)
              *reinterpret_cast<uint4*>(&v[q][p * 16 / sizeof(U)]) = __ldcs(reinterpret_cast<const uint4*>(row + c0) + p);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[q][e] = c0 + e < cols ? row[c0 + e] : SB::kOne;  // padding: bit 0 below
          }
        }
        if (++sg == spr) sg = 0, ++r;
      }
    }
#pragma unroll
    for (int q = 0; q < SEGS; ++q) {
      if (rr[q] >= rows) break;  // warp-uniform
      const I c0 = ss[q] * 256 + 8 * lane;
      uint32_t byte = 0;
      bool ok = true;
      if (sizeof(U) <= 4 && c0 + 8 <= cols) {
        // whole group, 32 bits at a time: validity as one masked compare per word, sign bits
        // gathered with shifts (per element, the loop below costs ~4x the instructions and made
        // the kernel issue-bound: fp16 and fp32 inputs packed in the same time)
        const uint32_t* w = reinterpret_cast<const uint32_t*>(v[q]);
        if constexpr (sizeof(U) == 2) {
          constexpr uint32_t kAbs2 = 0x7FFF7FFFu, kOne2 = ((uint32_t)SB::kOne << 16) | SB::kOne;
          ok = (((w[0] & kAbs2) ^ kOne2) | ((w[1] & kAbs2) ^ kOne2) | ((w[2] & kAbs2) ^ kOne2) |
                ((w[3] & kAbs2) ^ kOne2)) == 0u;
          // the sign bits are bit 7 of bytes 1 and 3 of every word: gather those bytes (elements 0-3,
          // 4-7), keep the negated sign bits, and one multiply moves bits 7/15/23/31 to 28-31
          const uint32_t lo = ~__byte_perm(w[0], w[1], 0x7531) & 0x80808080u;
          const uint32_t hi = ~__byte_perm(w[2], w[3], 0x7531) & 0x80808080u;
          byte = ((lo * 0x00204081u) >> 28) | (((hi * 0x00204081u) >> 28) << 4);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ok &= (w[i] & 0x7FFFFFFFu) == (uint32_t)SB::kOne;
            byte |= (~w[i] >> 31) << i;
          }
        }
      } else {
        ok = false;  // ragged tail / fp64: per element below
      }
      if (!ok) {
        byte = 0;
        int bad = -1;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool in = c0 + e < cols;
          if (in && (v[q][e] & SB::kAbs) != SB::kOne && bad < 0) bad = e;
          byte |= (uint32_t)(in && !(v[q][e] & SB::kSign)) << e;
        }
        if (bad >= 0) atomicMin(first_bad, (unsigned long long)((int64_t)rr[q] * cols + c0 + bad));
      }
      // word j of the segment = bytes of lanes 4j..4j+3
      const uint32_t b1 = __shfl_down_sync(0xffffffffu, byte, 1), b2 = __shfl_down_sync(0xffffffffu, byte, 2),
                     b3 = __shfl_down_sync(0xffffffffu, byte, 3);
      const I wj = ss[q] * 8 + (lane >> 2);
      if ((lane & 3) == 0 && wj < pitch) words[rr[q] * pitch + wj] = byte | (b1 << 8) | (b2 << 16) | (b3 << 24);
    }
  }
}

// ---- sign-of pack: bit = (v >= 0), the svid projection's np.where(Z >= 0, 1, -1) followed by
// pack (svid.py:99-103); no +-1 validation.
template <typename T>
__global__ void pack_sign_of_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols, int64_t ld,
                                    uint32_t* __restrict__ words, int64_t pitch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp >= rows * pitch) return;
  const int64_t r = warp / pitch, wj = warp % pitch;
  const int64_t c = wj * 32 + lane;
  const bool plus = c < cols && to_f64<T>(dense[r * ld + c]) >= 0.0;
  const uint32_t w = __ballot_sync(0xffffffffu, plus);
  if (lane == 0) words[r * pitch + wj] = w;
}

__global__ void init_first_bad_kernel(unsigned long long* p) { *p = ~0ull; }

// ---- unpack: the inverse of pack's layout -- a warp per 256-column segment (grid-stride); in each
// pass a lane expands the bits of its 16 bytes of output (8 fp16 / 4 fp32 / 2 fp64 columns) and
// writes them with one 16-byte store when its row is 16-byte aligned (a warp store = 512
// contiguous bytes); ragged tails element by element.
template <typename T> struct PlusMinus;
template <> struct PlusMinus<__half> { using U = uint16_t; static constexpr U kPlus = 0x3C00, kMinus = 0xBC00; };
template <> struct PlusMinus<__nv_bfloat16> { using U = uint16_t; static constexpr U kPlus = 0x3F80, kMinus = 0xBF80; };
template <> struct PlusMinus<float> { using U = uint32_t; static constexpr U kPlus = 0x3F800000u, kMinus = 0xBF800000u; };
template <> struct PlusMinus<double> {
  using U = unsigned long long;
  static constexpr U kPlus = 0x3FF0000000000000ull, kMinus = 0xBFF0000000000000ull;
};

template <typename T, typename I>  // I: index type, as pack_kernel
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t* __restrict__ words, I rows, I cols,
                                                     I pitch, T* __restrict__ dense, I ld, int vec_rows) {
  using PM = PlusMinus<T>;
  using U = typename PM::U;
  const int lane = threadIdx.x & 31;
  const I spr = (pitch + 7) / 8;
  const I nseg = rows * spr;
  const I nwarps = (I)(((int64_t)gridDim.x * blockDim.x) >> 5);
  for (I sgid = (I)((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5)); sgid < nseg; sgid += nwarps) {
    const I r = sgid / spr, sg = sgid - r * spr;
    U* row = reinterpret_cast<U*>(dense + r * ld);
    // E columns (16 bytes) per lane per pass, so each store instruction writes 512 contiguous bytes
    constexpr int E = 16 / (int)sizeof(U);
#pragma unroll
    for (int pass = 0; pass < 256 / (32 * E); ++pass) {
      const int o = pass * 32 * E + E * lane;  // column offset inside the segment
      const I c0 = sg * 256 + o;
      if (c0 >= cols) break;
      const uint32_t bits = __ldg(words + r * pitch + sg * 8 + (o >> 5)) >> (o & 31);
      U v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = ((bits >> e) & 1u) ? PM::kPlus : PM::kMinus;
      if (vec_rows && c0 + E <= cols) {
        __stcs(reinterpret_cast<uint4*>(row + c0), *reinterpret_cast<const uint4*>(v));
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (c0 + e < cols) row[c0 + e] = v[e];
      }
    }
  }
}

// ---- reference bytes (rows x ceil(cols/8)) -> canonical words; padding bits cleared.
__global__ void repack_u8_kernel(const uint8_t* __restrict__ bytes, int64_t rows, int64_t cols,
                                 uint32_t* __restrict__ words, int64_t pitch) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * pitch) return;
  const int64_t r = i / pitch, j = i % pitch;
  const int64_t rb = (cols + 7) >> 3;
  uint32_t w = 0;
  const int64_t c0 = j * 32;
  if (c0 < cols) {
    const uint8_t* row = bytes + r * rb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t bi = j * 4 + q;
      if (bi < rb) w |= (uint32_t)row[bi] << (8 * q);
    }
    const int64_t valid = cols - c0;
    if (valid < 32) w &= (1u << valid) - 1u;
  }
  words[i] = w;
}

// ---- canonical words -> reference bytes (padding bits of the last byte are zero).
__global__ void words_to_u8_kernel(const uint32_t* __restrict__ words, int64_t rows, int64_t cols,
                                   int64_t pitch, uint8_t* __restrict__ bytes) {
  const int64_t rb = (cols + 7) >> 3;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * rb) return;
  const int64_t r = i / rb, q = i % rb;
  uint32_t v = (__ldg(words + r * pitch + (q >> 2)) >> (8 * (q & 3))) & 0xffu;
  const int64_t valid = cols - q * 8;
  if (valid < 8) v &= (1u << valid) - 1u;
  bytes[i] = (uint8_t)v;
}

// ---- canonical words -> tiled decode layout.
// Output word (rb, c, lane, i), lane = 4*g + tig:
//   bit (8*b + r) <-> row 16*rb + g + 8*(i&1), column 256*c + 32*r + 4*tig + 16*(i>>1) + b.
// i.e. register a_i of the int8 m16n8k32 A fragment for k-block r is (word_i & (0x01010101<<r)):
// byte b of that register is column 4*tig+b (+16 for a2/a3) of row g (+8 for a1/a3), value
// 2^r when the sign is +1 and 0 when it is -1.
__global__ void tile_kernel(const uint32_t* __restrict__ words, int64_t rows, int64_t cols,
                            int64_t pitch, int64_t nchunks, uint32_t* __restrict__ tiled,
                            int64_t total_words) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= total_words) return;
  const int i = (int)(o & 3);
  const int lane = (int)((o >> 2) & 31);
  const int64_t blk = o >> 7;  // rb * nchunks + c
  const int64_t rb = blk / nchunks, c = blk % nchunks;
  const int g = lane >> 2, tig = lane & 3;
  const int64_t row = rb * 16 + g + 8 * (i & 1);
  uint32_t out = 0;
  if (row < rows) {
    const int base = 4 * tig + 16 * (i >> 1);
    const uint32_t* rw = words + row * pitch;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t wi = c * 8 + r;
      const uint32_t w = (wi < pitch) ? __ldg(rw + wi) : 0u;
      const uint32_t nib = (w >> base) & 0xfu;
      out |= ((nib & 1u) << r) | (((nib >> 1) & 1u) << (8 + r)) | (((nib >> 2) & 1u) << (16 + r)) |
             (((nib >> 3) & 1u) << (24 + r));
    }
  }
  tiled[o] = out;
}

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)ceil_div(n, threads); }

}  // namespace dbf

using namespace dbf;

// ---- canonical words -> paired prefill layout: per 32-column word, bit i (i < 16) holds column
// 2i and bit 16 + i holds column 2i + 1, so ONE shift brings the signs of the fp16 pair
// (2q, 2q+1) to bit positions 15 / 31 (prefill.cu).  Same pitch, padding bits stay zero.
__global__ void pair_kernel(const uint32_t* __restrict__ words, int64_t n, uint32_t* __restrict__ paired) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = words[i];
  uint32_t p = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) p |= ((c >> (2 * b)) & 1u) << b | ((c >> (2 * b + 1)) & 1u) << (16 + b);
  paired[i] = p;
}

// ---- bit-matrix transpose (canonical words): one warp per 32 x 32 bit block.  Lane i holds the
// word of row r0+i; __ballot_sync over bit j gives the word of transposed row c0+j (bit i <-> row
// r0+i).  Used for the transposed sign products of the staged gradients (budget.py:145-173,
// factorize.py:310-326): d_h2 = d_h3 @ A, d_h0 = (d_h2 * mid) @ B.
__global__ void transpose_kernel(const uint32_t* __restrict__ words, int64_t rows, int64_t cols, int64_t pitch,
                                 uint32_t* __restrict__ out, int64_t out_pitch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t rblocks = (rows + 31) >> 5, cblocks = (cols + 31) >> 5;
  if (warp >= rblocks * cblocks) return;
  const int64_t rb = warp % rblocks, cb = warp / rblocks;
  const int64_t r = rb * 32 + lane;
  const uint32_t w = (r < rows && cb < pitch) ? __ldg(words + r * pitch + cb) : 0u;
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const uint32_t t = __ballot_sync(0xffffffffu, (w >> j) & 1u);
    const int64_t orow = cb * 32 + j;
    if (lane == j && orow < cols) out[orow * out_pitch + rb] = t;
  }
}

// Zero the padding words of the transposed matrix (rows of out beyond the 32-bit blocks written).
__global__ void zero_pad_kernel(uint32_t* out, int64_t rows, int64_t pitch, int64_t first_word) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = pitch - first_word;
  if (per <= 0 || i >= rows * per) return;
  out[(i / per) * pitch + first_word + i % per] = 0u;
}

// ---- float64 sign GEMM on CUDA cores: out[i, r] = sum_c S[r, c] * x[i, c] (canonical words).
// The staged-gradient consumers (budget.channel_scores, factorize.refine_scales) are float64 numpy
// in the reference and their tests compare exact zeros / equalities (test_budget.py:97-104,
// test_factorize.py:231-238), so they get an fp64 path: one warp per (row, 4 input rows); lane =
// bit position, so the x loads of a 32-column word are one coalesced 256-byte access.
constexpr int kF64Batch = 4;
__global__ void sign_gemm_f64_kernel(const uint32_t* __restrict__ words, int64_t rows, int64_t cols, int64_t pitch,
                                     const double* __restrict__ x, int64_t ldx, int64_t batch,
                                     double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t bgroups = (batch + kF64Batch - 1) / kF64Batch;
  if (warp >= rows * bgroups) return;
  const int64_t r = warp / bgroups, i0 = (warp % bgroups) * kF64Batch;
  double acc[kF64Batch] = {0.0, 0.0, 0.0, 0.0};
  const int64_t nw = (cols + 31) >> 5;
  for (int64_t wi = 0; wi < nw; ++wi) {
    const uint32_t w = __ldg(words + r * pitch + wi);
    const int64_t c = wi * 32 + lane;
    if (c < cols) {
      const bool plus = (w >> lane) & 1u;
#pragma unroll
      for (int b = 0; b < kF64Batch; ++b)
        if (i0 + b < batch) {
          const double v = __ldg(x + (i0 + b) * ldx + c);
          acc[b] += plus ? v : -v;
        }
    }
  }
#pragma unroll
  for (int b = 0; b < kF64Batch; ++b) {
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o);
    if (lane == 0 && i0 + b < batch) out[(i0 + b) * ldo + r] = acc[b];
  }
}

extern "C" int dbf_pack_signs(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t ld,
                              uint32_t* words, int64_t word_pitch, int64_t* d_first_bad,
                              void* stream) {
  if (!dense || !words || !d_first_bad || rows < 1 || cols < 1 || ld < cols ||
      word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  auto* fb = reinterpret_cast<unsigned long long*>(d_first_bad);
  init_first_bad_kernel<<<1, 1, 0, s>>>(fb);
  return dispatch_float(dtype, [&](auto tag) {
    using T = decltype(tag);
    // rows start 16-byte aligned: every full 8-element group is one (fp16) or more 16-byte loads
    const int vec_rows = ((uintptr_t)dense & 15) == 0 && (ld * (int64_t)sizeof(T)) % 16 == 0;
    const int64_t groups = ceil_div(rows * ((word_pitch + 7) / 8), pack_segs<T>());
    // grid: 8 CTAs of 8 warps per SM (grid-stride), fewer when the matrix is small
    const int64_t blocks = std::min<int64_t>(ceil_div(groups, 8), (int64_t)kNumSMs * 8);
    const unsigned g = (unsigned)std::max<int64_t>(blocks, 1);
    if (rows * ld < INT32_MAX / 2 && rows * word_pitch < INT32_MAX / 2)
      pack_kernel<T, int><<<g, 256, 0, s>>>((const T*)dense, (int)rows, (int)cols, (int)ld, words, (int)word_pitch, fb,
                                            vec_rows);
    else
      pack_kernel<T, int64_t><<<g, 256, 0, s>>>((const T*)dense, rows, cols, ld, words, word_pitch, fb, vec_rows);
    return check_launch();
  });
}

extern "C" int dbf_unpack_signs(const uint32_t* words, int64_t rows, int64_t cols,
                                int64_t word_pitch, void* dense, int dtype, int64_t ld,
                                void* stream) {
  if (!dense || !words || rows < 1 || cols < 1 || ld < cols || word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  return dispatch_float(dtype, [&](auto tag) {
    using T = decltype(tag);
    const int vec_rows = ((uintptr_t)dense & 15) == 0 && (ld * (int64_t)sizeof(T)) % 16 == 0;
    const int64_t segs = rows * ((word_pitch + 7) / 8);
    const int64_t blocks = std::min<int64_t>(ceil_div(segs, 8), (int64_t)kNumSMs * 8);
    const unsigned g = (unsigned)std::max<int64_t>(blocks, 1);
    if (rows * ld < INT32_MAX / 2 && rows * word_pitch < INT32_MAX / 2)
      unpack_kernel<T, int><<<g, 256, 0, s>>>(words, (int)rows, (int)cols, (int)word_pitch, (T*)dense, (int)ld, vec_rows);
    else
      unpack_kernel<T, int64_t><<<g, 256, 0, s>>>(words, rows, cols, word_pitch, (T*)dense, ld, vec_rows);
    return check_launch();
  });
}

extern "C" int dbf_repack_u8(const uint8_t* bytes, int64_t rows, int64_t cols, uint32_t* words,
                             int64_t word_pitch, void* stream) {
  if (!bytes || !words || rows < 1 || cols < 1 || word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  repack_u8_kernel<<<grid_for(rows * word_pitch, 256), 256, 0, (cudaStream_t)stream>>>(
      bytes, rows, cols, words, word_pitch);
  return check_launch();
}

extern "C" int dbf_words_to_u8(const uint32_t* words, int64_t rows, int64_t cols,
                               int64_t word_pitch, uint8_t* bytes, void* stream) {
  if (!bytes || !words || rows < 1 || cols < 1 || word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  const int64_t n = rows * ((cols + 7) >> 3);
  words_to_u8_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(words, rows, cols,
                                                                         word_pitch, bytes);
  return check_launch();
}

extern "C" int dbf_tile_signs(const uint32_t* words, int64_t rows, int64_t cols,
                              int64_t word_pitch, void* tiled, void* stream) {
  if (!tiled || !words || rows < 1 || cols < 1 || word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  const int64_t nch = chunks(cols);
  const int64_t total = row_blocks(rows) * nch * (kChunkBytes / 4);
  tile_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      words, rows, cols, word_pitch, nch, (uint32_t*)tiled, total);
  return check_launch();
}

extern "C" int dbf_pair_signs(const uint32_t* words, int64_t rows, int64_t word_pitch, uint32_t* paired,
                              void* stream) {
  if (!words || !paired || rows < 1 || word_pitch < 1) return DBF_ERR_INVALID_ARGUMENT;
  const int64_t n = rows * word_pitch;
  pair_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(words, n, paired);
  return check_launch();
}

extern "C" int dbf_transpose_signs(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                                   uint32_t* out, int64_t out_pitch, void* stream) {
  if (!words || !out || rows < 1 || cols < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (word_pitch < ceil_div(cols, 32) || out_pitch < ceil_div(rows, 32)) return DBF_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nwarps = ceil_div(rows, 32) * ceil_div(cols, 32);
  transpose_kernel<<<(unsigned)ceil_div(nwarps * 32, 256), 256, 0, s>>>(words, rows, cols, word_pitch, out,
                                                                         out_pitch);
  int st = check_launch();
  if (st != DBF_OK) return st;
  const int64_t first = ceil_div(rows, 32);
  if (out_pitch > first) {
    const int64_t n = cols * (out_pitch - first);
    zero_pad_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(out, cols, out_pitch, first);
    st = check_launch();
  }
  return st;
}

extern "C" int dbf_sign_gemm_f64(const uint32_t* words, int64_t rows, int64_t cols, int64_t word_pitch,
                                 const double* x, int64_t ldx, int64_t batch, double* out, int64_t ldo,
                                 void* stream) {
  if (!words || !x || !out || rows < 1 || cols < 1 || batch < 1) return DBF_ERR_INVALID_ARGUMENT;
  if (word_pitch < ceil_div(cols, 32) || ldx < cols || ldo < rows) return DBF_ERR_SHAPE;
  const int64_t nwarps = rows * ceil_div(batch, kF64Batch);
  sign_gemm_f64_kernel<<<(unsigned)ceil_div(nwarps * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      words, rows, cols, word_pitch, x, ldx, batch, out, ldo);
  return check_launch();
}

extern "C" int dbf_pack_sign_of(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t ld,
                                uint32_t* words, int64_t word_pitch, void* stream) {
  if (!dense || !words || rows < 1 || cols < 1 || ld < cols || word_pitch < canonical_pitch(cols))
    return DBF_ERR_INVALID_ARGUMENT;
  const int64_t threads = rows * word_pitch * 32;
  return dispatch_float(dtype, [&](auto tag) {
    using T = decltype(tag);
    pack_sign_of_kernel<T><<<grid_for(threads, 256), 256, 0, (cudaStream_t)stream>>>((const T*)dense, rows, cols,
                                                                                        ld, words, word_pitch);
    return check_launch();
  });
}
