// Microbenchmark: latency of the decode engine's per-chunk input loads on B200.
// 148 CTAs x 16 warps; each warp repeatedly loads one 256-column chunk (lane: 2 x 8-byte fp16
// groups + 2 x 8-byte scale groups) of an L2-resident vector and reduces it with shuffles, the
// way quantize does.  Variants: ld.global.nc (__ldg), ld.relaxed.gpu, ld.global (default),
// and with a concurrent cp.async.bulk weight stream from HBM on a producer warp.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint2 ld_relaxed(const void* p) {
  uint2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(544, 1) lat(const __half* x, const __half* sc, int cols, int iters, long long* out,
                                             const uint8_t* wsrc, size_t wbytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  if (warp == 16) {
    if (MODE >= 3 && lane == 0) {  // stream weights: 16 KB bulk copies, one at a time
      uint32_t ph = 0;
      for (int i = 0; i < iters * 4; ++i) {
        const uint8_t* src = wsrc + ((size_t)(blockIdx.x * 997 + i) * 16384) % (wbytes - 16384);
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16384) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(smem)),
                     "l"(src), "r"(b)
                     : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(b),
                     "r"(ph)
                     : "memory");
        ph ^= 1;
      }
    }
    return;
  }
  long long tot = 0;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int c = (blockIdx.x * 16 + warp + it * 7) % (cols / 256);
    const int c0 = c * 256;
    const long long t0 = clock64();
    uint2 v0, v1, s0, s1;
    const int j0 = c0 + 4 * lane, j1 = c0 + 4 * (lane + 32);
    if (MODE == 0 || MODE == 3) {
      v0 = __ldg((const uint2*)(x + j0)); v1 = __ldg((const uint2*)(x + j1));
      s0 = __ldg((const uint2*)(sc + j0)); s1 = __ldg((const uint2*)(sc + j1));
    } else if (MODE == 1 || MODE == 4) {
      v0 = ld_relaxed(x + j0); v1 = ld_relaxed(x + j1);
      s0 = ld_relaxed(sc + j0); s1 = ld_relaxed(sc + j1);
    } else {
      v0 = *(const uint2*)(x + j0); v1 = *(const uint2*)(x + j1);
      s0 = *(const uint2*)(sc + j0); s1 = *(const uint2*)(sc + j1);
    }
    float m = fabsf(__low2float(*(__half2*)&v0.x) * __low2float(*(__half2*)&s0.x)) +
              fabsf(__high2float(*(__half2*)&v1.y) * __high2float(*(__half2*)&s1.y));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const long long t1 = clock64();
    tot += t1 - t0;
    acc += m;
  }
  if (lane == 0) out[blockIdx.x * 16 + warp] = tot / iters + (acc == 12345.f);
}

int main() {
  const int cols = 11008, iters = 200;
  __half *x, *sc;
  cudaMalloc(&x, cols * 2);
  cudaMalloc(&sc, cols * 2);
  cudaMemset(x, 0, cols * 2);
  cudaMemset(sc, 0, cols * 2);
  const size_t wbytes = (size_t)1 << 30;
  uint8_t* w;
  cudaMalloc(&w, wbytes);
  cudaMemset(w, 1, wbytes);
  long long* d;
  cudaMalloc(&d, 148 * 16 * 8);
  static long long h[148 * 16];
  const char* names[] = {"ld.global.nc", "ld.relaxed.gpu", "ld.global", "ld.global.nc + weight stream",
                         "ld.relaxed.gpu + weight stream"};
  void (*ks[])(const __half*, const __half*, int, int, long long*, const uint8_t*, size_t) = {
      lat<0>, lat<1>, lat<2>, lat<3>, lat<4>};
  for (int k = 0; k < 5; ++k) {
    cudaFuncSetAttribute(ks[k], cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    ks[k]<<<148, 544, 64 * 1024>>>(x, sc, cols, iters, d, w, wbytes);
    ks[k]<<<148, 544, 64 * 1024>>>(x, sc, cols, iters, d, w, wbytes);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148 * 16; ++i) avg += h[i];
    printf("%-34s %s  cycles per chunk load+reduce: %.0f\n", names[k], cudaGetErrorString(e), avg / (148 * 16));
  }
  return 0;
}
