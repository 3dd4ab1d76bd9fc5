// Cost of reading %globaltimer and its granularity, measured with clock64 (one warp).
#include <cstdio>
__global__ void k(long long* out) {
  long long t0 = clock64(), g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  long long t2 = clock64();
  long long gmin = 1ll << 60, prev = g1;
  for (int i = 0; i < 1000; ++i) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (g != prev && g - prev < gmin) gmin = g - prev;
    prev = g;
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = g1 - g0; out[3] = gmin; out[4] = (t3 - t2) / 1000; }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[5];
  for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(d); cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost); }
  printf("globaltimer read: %lld / %lld cycles, delta %lld ns, granularity %lld ns, loop %lld cyc/read\n", h[0], h[1], h[2], h[3], h[4]);
}
