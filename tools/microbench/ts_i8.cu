// Microbenchmark + layout check for an int8 tensor-memory decode path on B200 (sm_100a):
//  1. tcgen05.mma.kind::i8, A (128 x 32 s8) from TMEM, B (16 x 32 s8, K-major, no swizzle) from
//     shared memory, D s32 in TMEM: checks the result against a CPU product for both readings of
//     the no-swizzle LBO/SBO fields;
//  2. issue rate of back-to-back M=128 N=16 K=32 i8 MMAs from one thread;
//  3. tcgen05.st throughput (32x32b.x8 / x16) with 4, 8 and 16 warps per SM, all 148 SMs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../paper_2505_11076_b200/csrc/sm100.cuh"

using namespace dbf::sm100;

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                     // D: s32
         | (1u << 7) | (1u << 10)      // A, B: signed 8-bit
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t sdesc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1u << 46);
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// A: 128 x 32 s8 row-major; B: 16 x 32 s8 row-major (row = n); out: 128 x 16 s32
__global__ void check_kernel(const int8_t* A, const int8_t* B, int* out, int variant, long long* cyc, int reps,
                             int N = 16, int nacc = 1) {
  __shared__ __align__(1024) int8_t bs[256 * 32];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B in the canonical no-swizzle K-major layout: core matrix = 8 rows x 16 B;
  // element (n, k) at (n / 8) * SBO_mn + (k / 16) * LBO_k + (n % 8) * 16 + k % 16
  const uint32_t stride_k = variant == 0 ? 128 : 256, stride_mn = variant == 0 ? 256 : 128;
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32;
    bs[(n / 8) * stride_mn + (k / 16) * stride_k + (n % 8) * 16 + k % 16] = B[i];
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = taddr_s;
  // A into TMEM columns 32..39: lane = row, column j = k 4j..4j+3 (little-endian bytes)
  {
    const int row = warp * 32 + lane;
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = *(const uint32_t*)(A + row * 32 + 4 * j);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tm + ((uint32_t)(warp * 32) << 16) + 32),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t bd = sdesc_none(smem_u32(bs), variant == 0 ? 128 : 256, variant == 0 ? 256 : 128);
    const long long t0 = clock64();
    if (N == 16 && nacc == 1) {
      for (int r = 0; r < reps; ++r) mma_i8_ts(tm, tm + 32, bd, idesc_i8(128, 16), r > 0 ? 1u : 0u);
    } else {
      // nacc accumulators (columns 256 + j * N) and A tiles rotating over columns 32..223
      const uint32_t id = idesc_i8(128, N);
      for (int r = 0; r < reps; ++r)
        mma_i8_ts(tm + 256 + (uint32_t)(((r % nacc) * N) % 256), tm + 32 + (uint32_t)((r * 8) % 192), bd, id,
                  r >= nacc ? 1u : 0u);
    }
    const long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t0;
  }
  __syncthreads();
  tc_fence_after();
  {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tm + ((uint32_t)(warp * 32) << 16)));
    tmem_wait_ld();
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) out[row * 16 + j] = (int)v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int X>
__global__ void st_kernel(int iters, long long* out) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = taddr_s;
  const int nw = blockDim.x >> 5;
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * (512 / (nw / 4)));
  uint32_t v[16];
  for (int j = 0; j < 16; ++j) v[j] = lane * 16 + j;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t a = base + (uint32_t)((i * X) % (512 / (nw / 4)));
    if (X == 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
    else
      tmem_st16(a, v);
    if ((i & 3) == 3) tmem_wait_st();
    v[0] += 1;
  }
  tmem_wait_st();
  const long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  int8_t hA[128 * 32], hB[16 * 32];
  srand(1);
  for (auto& a : hA) a = (int8_t)(rand() % 256 - 128);
  for (auto& b : hB) b = (int8_t)(rand() % 256 - 128);
  int ref[128 * 16];
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      int s = 0;
      for (int k = 0; k < 32; ++k) s += hA[m * 32 + k] * hB[n * 32 + k];
      ref[m * 16 + n] = s;
    }
  int8_t *dA, *dB;
  int* dO;
  long long* dc;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dO, 128 * 16 * 4);
  cudaMalloc(&dc, 148 * 32 * 8);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    check_kernel<<<1, 128>>>(dA, dB, dO, variant, dc, 1);
    cudaError_t e = cudaDeviceSynchronize();
    int h[128 * 16];
    cudaMemcpy(h, dO, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * 16; ++i) bad += h[i] != ref[i];
    printf("i8 TS MMA layout variant %d (K-dir stride %d): %s, mismatches %d / 2048 (h[0]=%d ref=%d)\n", variant,
           variant == 0 ? 128 : 256, cudaGetErrorString(e), bad, h[0], ref[0]);
  }
  for (int reps : {64, 1024}) {
    check_kernel<<<1, 128>>>(dA, dB, dO, 0, dc, reps);
    cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("i8 MMA M128 N16 K32 x%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", reps, (double)c[0] / reps,
           (double)c[1] / reps);
  }
  for (int N : {16, 32, 64, 128, 256})
    for (int nacc : {1, 4}) {
      if (N * nacc > 256) continue;
      const int reps = 1024;
      check_kernel<<<1, 128>>>(dA, dB, dO, 0, dc, reps, N, nacc);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[2];
      cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
      printf("i8 MMA M128 N%-3d K32, %d accumulators, rotating A: %s issue %.1f complete %.1f cyc/mma\n", N, nacc,
             cudaGetErrorString(e), (double)c[0] / reps, (double)c[1] / reps);
    }
  for (int nw : {4, 8, 16}) {
    for (int x : {8, 16}) {
      const int iters = 4096;
      if (x == 8) st_kernel<8><<<148, nw * 32>>>(iters, dc);
      else st_kernel<16><<<148, nw * 32>>>(iters, dc);
      cudaError_t e = cudaDeviceSynchronize();
      static long long h[148 * 32];
      cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int b = 0; b < 148; ++b)
        for (int w = 0; w < nw; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
      const double bytes = (double)nw * iters * 32 * x * 4;
      printf("tcgen05.st x%-2d %2d warps: %s  %.1f B/clk/SM\n", x, nw, cudaGetErrorString(e), bytes / mx);
    }
  }
  return 0;
}
