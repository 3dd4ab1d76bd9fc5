// Microbenchmark: TMA 2-D box throughput per SM by ISSUER LAYOUT (B200).  148 CTAs, one per SM;
// fp16 activations T x K with 128-byte swizzled boxes of 64 columns x R rows (the prefill kernel's
// activation boxes).  Each issuer keeps S boxes in flight (waits on its oldest before issuing).
//   mode 0: P issuers = lane 0 of P different warps
//   mode 1: P issuers = lanes 0..P-1 of ONE warp (divergent mbarrier waits, the round-2 prefill)
//   mode 2: ONE thread, P*S boxes in flight
// Question: is the prefill's ~600-780 cycles per box a TMA limit or an issue-layout artifact?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_11076_b200/csrc tma_issue.cu -o tma_issue -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace dbf::sm100;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int kMaxSlots = 24;

__global__ void __launch_bounds__(384, 1)
    bench(const __grid_constant__ CUtensorMap map, int R, int S, int P, int mode, int nk, int ntok, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kMaxSlots];
  const int box_bytes = R * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slots = P * S;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int id = -1, nid = P, per = S;
  if (mode == 0 && lane == 0 && warp < P) id = warp;
  if (mode == 1 && warp == 0 && lane < P) id = lane;
  if (mode == 2 && threadIdx.x == 0) id = 0, nid = 1, per = slots;
  const int tok0 = (blockIdx.x % ntok) * R;
  long long t0 = clock64();
  if (id >= 0) {
    const uint64_t pol = policy_evict_last();
    int cnt = 0;
    for (int kb = id; kb < nk; kb += nid, ++cnt) {
      const int s = id * per + cnt % per;
      if (cnt >= per) mbar_wait(&full[s], ((cnt - per) / per) & 1);
      mbar_arrive_expect_tx(&full[s], box_bytes);
      tma_load_2d(smem + (size_t)s * box_bytes, &map, kb * 64, tok0, &full[s], pol);
    }
    for (int j = (cnt > per ? cnt - per : 0); j < cnt; ++j) mbar_wait(&full[id * per + j % per], (j / per) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

__global__ void fill_random(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = x & 0x3BFF3BFFu;
  }
}

int main() {
  const int T = 2048, K = 16384;  // 64 MB: L2-resident like the prefill's activations
  void* x;
  cudaMalloc(&x, (size_t)T * K * 2);
  fill_random<<<1024, 256>>>((uint32_t*)x, (size_t)T * K / 2);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeTiledFn fn = (EncodeTiledFn)fnp;
  const int smem = 220 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Cfg { int R, S, P, mode; };
  const Cfg cfgs[] = {
      {256, 6, 1, 2}, {256, 2, 3, 0}, {256, 2, 3, 1}, {256, 1, 6, 0}, {256, 1, 6, 1},
      {128, 12, 1, 2}, {128, 4, 3, 0}, {128, 4, 3, 1}, {128, 1, 12, 0}, {128, 1, 12, 1}, {128, 2, 6, 0},
      {64, 12, 1, 2}, {64, 4, 3, 1}, {64, 4, 3, 0}, {64, 24, 1, 2},
  };
  for (const Cfg& c : cfgs) {
    if ((size_t)c.S * c.P * c.R * 128 + 1024 > (size_t)smem || c.S * c.P > kMaxSlots) { printf("skip\n"); continue; }
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)c.R};
    const cuuint32_t estr[2] = {1, 1};
    fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nk = K / 64;
    for (int rep = 0; rep < 3; ++rep) bench<<<148, 384, smem>>>(map, c.R, c.S, c.P, c.mode, nk, T / c.R, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("box 64x%-3d mode %d (%s) P %2d S %2d in flight %2d: %s  %6.0f cycles/box  %5.1f B/clk/SM\n", c.R, c.mode,
           c.mode == 0 ? "warps" : c.mode == 1 ? "lanes" : "1 thr", c.P, c.S, c.P * c.S, cudaGetErrorString(e),
           avg / nk, (double)nk * c.R * 128 / avg);
  }
  return 0;
}
