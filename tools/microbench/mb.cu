// Microbenchmarks that size the DBF decode design on B200 (sm_100a).
// 1) IMMA m16n8k32 s8 and HMMA m16n8k16 throughput (mma.sync, register operands)
// 2) sign-expansion loop: 1 LOP3 per 4 weights + IMMA (the decode inner loop, from registers)
// 3) cross-CTA flag hop latency (st.release / ld.acquire ping-pong between two CTAs)
// 4) HBM streaming read bandwidth (LDG.128, grid = k*148)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ void imma(int* c, uint32_t a0,uint32_t a1,uint32_t a2,uint32_t a3,uint32_t b0,uint32_t b1){
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
   : "+r"(c[0]),"+r"(c[1]),"+r"(c[2]),"+r"(c[3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
}
__device__ __forceinline__ void hmma(float* c, uint32_t a0,uint32_t a1,uint32_t a2,uint32_t a3,uint32_t b0,uint32_t b1){
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
   : "+f"(c[0]),"+f"(c[1]),"+f"(c[2]),"+f"(c[3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
}

__global__ void k_imma(int iters, int* out, uint32_t seed){
  int c[8][4] = {};
  uint32_t a = seed ^ threadIdx.x, b = seed * 7 + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) imma(c[j], a, a+j, a^j, a|j, b, b+j);
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0]+c[j][1]+c[j][2]+c[j][3];
  out[blockIdx.x*blockDim.x+threadIdx.x] = s;
}
__global__ void k_hmma(int iters, float* out, uint32_t seed){
  float c[8][4] = {};
  uint32_t a = 0x3c003c00u ^ (threadIdx.x & 1), b = 0x3c00bc00u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hmma(c[j], a, a, a, a, b, b);
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0]+c[j][1]+c[j][2]+c[j][3];
  out[blockIdx.x*blockDim.x+threadIdx.x] = s;
}
// expansion loop: per 4 words (128 sign bits per lane) -> 32 LOP3 + 8 IMMA, B fragments from registers
__global__ void k_expand(int iters, int* out, uint32_t seed){
  int c[4] = {};
  uint32_t w0 = seed ^ threadIdx.x, w1 = w0*3u, w2 = w0*5u, w3 = w0*9u;
  uint32_t b[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) b[j] = seed + j*threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      uint32_t m = 0x01010101u << r;
      imma(c, w0 & m, w1 & m, w2 & m, w3 & m, b[2*r], b[2*r+1]);
    }
    w0 = w0 * 1664525u + 1013904223u; w1 ^= w0; w2 += w1; w3 ^= w2;   // fresh words (4 int ops ~ a load)
  }
  out[blockIdx.x*blockDim.x+threadIdx.x] = c[0]+c[1]+c[2]+c[3];
}
// flag ping-pong between CTA 0 and CTA 1 (on different SMs)
__global__ void k_pingpong(int rounds, unsigned* flags, long long* cycles){
  unsigned* mine = flags + (blockIdx.x ? 32 : 0);
  unsigned* other = flags + (blockIdx.x ? 0 : 32);
  if (threadIdx.x) return;
  long long t0 = clock64();
  for (int i = 1; i <= rounds; ++i) {
    if (blockIdx.x == 0) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(mine), "r"(i) : "memory");
      unsigned v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(other) : "memory"); } while (v < (unsigned)i);
    } else {
      unsigned v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(other) : "memory"); } while (v < (unsigned)i);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(mine), "r"(i) : "memory");
    }
  }
  cycles[blockIdx.x] = clock64() - t0;
}
// relaxed variant (plain volatile st / ld, no fences) = LL-protocol style
__global__ void k_pingpong_relaxed(int rounds, unsigned* flags, long long* cycles){
  volatile unsigned* mine = flags + (blockIdx.x ? 32 : 0);
  volatile unsigned* other = flags + (blockIdx.x ? 0 : 32);
  if (threadIdx.x) return;
  long long t0 = clock64();
  for (int i = 1; i <= rounds; ++i) {
    if (blockIdx.x == 0) { *mine = i; while (*other < (unsigned)i) {} }
    else { while (*other < (unsigned)i) {} *mine = i; }
  }
  cycles[blockIdx.x] = clock64() - t0;
}
__global__ void k_stream(const int4* __restrict__ p, size_t n, int* out){
  int4 acc = make_int4(0,0,0,0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride*4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i + u*stride < n) ? __ldg(p + i + u*stride) : make_int4(0,0,0,0);
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) out[0] = 1;
}

int main(){
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d MB clock(attr) %d MHz\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, clk_khz/1000);
  int nsm = pr.multiProcessorCount;
  int* dout; CK(cudaMalloc(&dout, 64<<20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int warps : {4, 8, 16}) {
    int iters = 4096; dim3 g(nsm*2), b(32*warps);
    k_imma<<<g,b>>>(16, dout, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_imma<<<g,b>>>(iters, dout, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)g.x*warps*iters*8;
    printf("IMMA.16832 u8.s8: warps/CTA=%d (2 CTA/SM)  %.1f G mma/s  = %.1f int8 TOPS dense  (%.3f ms)\n", warps, mmas/ms/1e6, mmas*4096*2/ms/1e9, ms);
    k_hmma<<<g,b>>>(16, (float*)dout, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_hmma<<<g,b>>>(iters, (float*)dout, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("HMMA.16816 f16->f32: warps/CTA=%d  %.1f G mma/s = %.1f TFLOPS dense\n", warps, mmas/ms/1e6, mmas*2048*2/ms/1e9);
    k_expand<<<g,b>>>(16, dout, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_expand<<<g,b>>>(iters, dout, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double elems = (double)g.x*warps*32*iters*128;
    printf("expand(LOP3+IMMA) : warps/CTA=%d  %.1f T sign-elem/s = %.0f GB/s of packed signs\n", warps, elems/ms/1e9, elems/8/ms/1e6);
  }
  unsigned* flags; CK(cudaMalloc(&flags, 4096)); long long* cyc; CK(cudaMalloc(&cyc, 64));
  for (int variant = 0; variant < 2; ++variant) for (int far : {1, 74, 100}) {
    CK(cudaMemset(flags, 0, 4096));
    // launch nsm CTAs so CTA 0 and CTA 'far' land on distinct SMs; only blocks 0 and 1 participate: use grid 2 with big smem to force separate SMs
    int rounds = 2000;
    cudaFuncSetAttribute(k_pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
    cudaFuncSetAttribute(k_pingpong_relaxed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
    cudaEventRecord(e0);
    if (variant == 0) k_pingpong<<<2, 32, 200*1024>>>(rounds, flags, cyc);
    else k_pingpong_relaxed<<<2, 32, 200*1024>>>(rounds, flags, cyc);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("flag ping-pong (%s): %.0f ns per one-way hop\n", variant ? "volatile" : "release/acquire", ms*1e6/rounds/2);
    break;
  }
  size_t bytes = (size_t)2 << 30; int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  for (int mult : {1, 2, 4, 8}) {
    dim3 g(nsm*mult), b(512);
    k_stream<<<g,b>>>(buf, bytes/16, dout); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_stream<<<g,b>>>(buf, bytes/16, dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 stream read: grid=%d x512  %.0f GB/s\n", g.x, 5.0*bytes/ms/1e6);
  }
  // small-kernel latency: empty-ish kernel back to back
  cudaEventRecord(e0); for (int r = 0; r < 1000; ++r) k_stream<<<nsm,512>>>(buf, 0, dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel back-to-back: %.2f us per launch\n", ms);
  CK(cudaGetLastError());
  return 0;
}
