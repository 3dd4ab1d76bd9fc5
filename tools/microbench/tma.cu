// Microbenchmark: TMA 2-D tile load throughput per SM on B200 (fp16, 128-byte swizzle boxes of 64 x R),
// one producer thread per CTA keeping S tiles in flight; 148 CTAs.  Tiles are read from a T x K fp16
// activation matrix; `share` CTAs walk the same tile sequence (the prefill kernel's re-read pattern).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace dbf::sm100;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void __launch_bounds__(1024, 1)
    tma_bench(const __grid_constant__ CUtensorMap map, int rows_box, int stages, int nk, int ntok_tiles, int share,
              long long* out, int nprod, int hint, const void* x_raw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[4][16];
  const int tile_bytes = rows_box * 128;
  const int pw = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; ++w)
      for (int i = 0; i < stages; ++i) mbar_init(&full[w][i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && pw < nprod) {
    const int tok_tile = (blockIdx.x / share) % ntok_tiles;
    const uint64_t pol = policy_evict_last();
    uint8_t* mysmem = smem + (size_t)pw * stages * tile_bytes;
    long long t0 = clock64();
    int cnt = 0;
    for (int kb = pw; kb < nk + stages * nprod; kb += nprod, ++cnt) {
      if (cnt >= stages) {
        const int j = cnt - stages;
        mbar_wait(&full[pw][j % stages], (j / stages) & 1);
      }
      if (kb < nk) {
        const int s = cnt % stages;
        mbar_arrive_expect_tx(&full[pw][s], tile_bytes);
        if (hint == 2) {
          // 1-D bulk copy of a contiguous tile (the tiled-activation alternative)
          const char* src = (const char*)x_raw + ((size_t)tok_tile * nk + kb) * tile_bytes;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(mysmem + (size_t)s * tile_bytes)),
              "l"(src), "r"(tile_bytes), "r"(smem_u32(&full[pw][s]))
              : "memory");
        } else if (hint)
          tma_load_2d(mysmem + (size_t)s * tile_bytes, &map, kb * 64, tok_tile * rows_box, &full[pw][s], pol);
        else
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  smem_u32(mysmem + (size_t)s * tile_bytes)),
              "l"(&map), "r"(kb * 64), "r"(tok_tile * rows_box), "r"(smem_u32(&full[pw][s]))
              : "memory");
      }
    }
    if (pw == 0) out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
}

__global__ void fill_random(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = x & 0x3BFF3BFFu;  // finite fp16 pairs
  }
}

int main(int argc, char** argv) {
  const int T = 2048, K = 4096;
  void* x;
  cudaMalloc(&x, (size_t)T * K * 2);
  cudaMemset(x, 0, (size_t)T * K * 2);
  if (argc > 1) { fill_random<<<1024, 256>>>((uint32_t*)x, (size_t)T * K / 2); cudaDeviceSynchronize(); printf("random data\n"); }
  long long* d;
  cudaMalloc(&d, 148 * 8);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeTiledFn fn = (EncodeTiledFn)fnp;
  cudaFuncSetAttribute(tma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int threads = argc > 2 ? atoi(argv[2]) : 128;
  const int smem_dyn = (argc > 3 ? atoi(argv[3]) : 200) * 1024;
  printf("threads %d smem %d\n", threads, smem_dyn);
  struct Cfg { int R, S, share, nprod, hint, swz; };
  const Cfg cfgs[] = {{128, 4, 8, 1, 1, 1}, {128, 2, 8, 2, 1, 1}, {128, 2, 8, 4, 1, 1},
                      {128, 4, 8, 1, 2, 1}, {128, 8, 8, 1, 2, 1}, {128, 2, 8, 4, 2, 1}, {256, 4, 8, 1, 2, 1}};
  for (const Cfg& c : cfgs) {
    const int R = c.R, S = c.S, share = c.share;
    if ((size_t)S * c.nprod * R * 128 + 2048 > (size_t)smem_dyn) { printf("skip (smem)\n"); continue; }
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)R};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
       c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nk = K / 64;
    for (int rep = 0; rep < 2; ++rep)
      tma_bench<<<148, threads, smem_dyn>>>(map, R, S, nk, T / R, share, d, c.nprod, c.hint, x);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double bpc = (double)nk * R * 128 / avg;
    printf("box 64x%d stages %d share %2d nprod %d hint %d swz %d: %s/%d  %.0f cycles/tile  %.1f B/clk/SM  (x148 = %.0f B/clk)\n",
           R, S, share, c.nprod, c.hint, c.swz, cudaGetErrorString(e), (int)cr, avg / nk, bpc, bpc * 148);
  }
  return 0;
}
