// Ring microbenchmark: one producer lane streams `piece` bytes per cp.async.bulk into a shared
// ring of `slots` slots; 15 consumer warps wait/release each slot (optionally running the
// int8 sign-GEMV inner loop on it).  Reports GB/s over a 2 GB stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c){asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(sa(b)),"r"(c));}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n){asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"::"r"(sa(b)),"r"(n):"memory");}
__device__ __forceinline__ void mbar_arrive(uint64_t* b){asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];"::"r"(sa(b)):"memory");}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph){asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}"::"r"(sa(b)),"r"(ph):"memory");}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b){asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(d)),"l"(s),"r"(n),"r"(sa(b)):"memory");}
__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0,uint32_t a1,uint32_t a2,uint32_t a3,uint32_t b0,uint32_t b1){
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
   : "+r"(c[0]),"+r"(c[1]),"+r"(c[2]),"+r"(c[3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));}
template <int MODE, int W>
__global__ void __launch_bounds__(512,1) ring(const uint8_t* src, size_t per_cta, int piece, int slots, int* out){
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + slots*piece); uint64_t* empty = full + 32;
  uint8_t* xf = (uint8_t*)(empty + 32);
  int warp = threadIdx.x>>5, lane = threadIdx.x&31;
  if (threadIdx.x==0){ for(int i=0;i<slots;++i){mbar_init(&full[i],1); mbar_init(&empty[i],W);} asm volatile("fence.mbarrier_init.release.cluster;":::"memory"); }
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) xf[i] = i*7;
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta;
  int npieces = per_cta / piece;
  if (warp == W) {
    if (lane == 0) { int s=0; uint32_t ph=0;
      for (int p=0;p<npieces;++p){ mbar_wait(&empty[s], ph^1); mbar_expect(&full[s], piece); bulk(sm + s*piece, base + (size_t)p*piece, piece, &full[s]); if(++s==slots){s=0;ph^=1;} } }
    return;
  }
  int s=0; uint32_t ph=0; int acc[4][4] = {}; int acc8[8][4] = {}; uint32_t x = 0;
  uint2 bb[8];
  for (int r = 0; r < 8; ++r) bb[r] = make_uint2(0, 0);
  const int nch = piece/512; int cb = 0;
  for (int p=0;p<npieces;++p){
    mbar_wait(&full[s], ph);
    if (MODE == 6) {
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece) + lane;
      const uint2* xb = (const uint2*)xf + (lane & 15);
      const bool lo = lane < 16;
      for (int c = first; c < nch; c += W) {
        const uint4 w = pc[c*32];
        const uint2* xk = xb + ((c*8) & 31) * 16;
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r; if (lo) bb[r] = xk[r*16];
          imma(acc[r&3], w.x&m, w.y&m, w.z&m, w.w&m, bb[r].x, bb[r].y); }
      }
      cb += nch;
    } else if (MODE == 7) {
      // two row blocks per iteration share each B fragment (piece = 2 units of nch/2 chunks)
      const int half = nch / 2;
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece) + lane;
      const uint2* xb = (const uint2*)xf + (lane & 15);
      const bool lo = lane < 16;
      for (int c = first; c < half; c += W) {
        const uint4 w0 = pc[c*32], w1 = pc[(c+half)*32];
        const uint2* xk = xb + ((c*8) & 31) * 16;
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r; if (lo) bb[r] = xk[r*16];
          imma(acc[r&1], w0.x&m, w0.y&m, w0.z&m, w0.w&m, bb[r].x, bb[r].y);
          imma(acc[2+(r&1)], w1.x&m, w1.y&m, w1.z&m, w1.w&m, bb[r].x, bb[r].y); }
      }
      cb += half;
    } else if (MODE == 4 || MODE == 5) {
      // predicated (lanes 0-15) B loads without zeroing, 8 accumulator chains, prefetched weights
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece) + lane;
      const uint32_t xb = sa((const uint2*)xf + (lane & 15));
      const bool lo = lane < 16;
      int c = first;
      uint4 w = c < nch ? pc[c*32] : make_uint4(0,0,0,0);
      for (; c < nch; c += W) {
        const uint4 wn = (c + W < nch) ? pc[(c+W)*32] : make_uint4(0,0,0,0);
        const uint32_t xk = xb + ((c*8) & 31) * 128;
        uint32_t b0[8], b1[8];
#pragma unroll
        for (int r=0;r<8;++r) asm volatile("{.reg .pred p; setp.ne.b32 p, %2, 0; @p ld.shared.v2.u32 {%0,%1}, [%3];}" : "+r"(b0[r]), "+r"(b1[r]) : "r"((int)lo), "r"(xk + r*128));
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r;
          if (MODE == 4) imma(acc8[r], w.x&m, w.y&m, w.z&m, w.w&m, b0[r], b1[r]);
          else imma(acc[r&3], w.x&m, w.y&m, w.z&m, w.w&m, b0[r], b1[r]); }
        w = wn;
      }
      cb += nch;
    } else if (MODE == 3) {
      // lean: unpredicated B-fragment loads (lanes 16-31 duplicate lanes 0-15), immediate offsets
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece) + lane;
      const uint2* xb = (const uint2*)xf + (lane & 15);
      for (int c = first; c < nch; c += W) {
        const uint4 w = pc[c*32];
        const uint2* xk = xb + ((c*8) & 31) * 16;
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r; const uint2 b = xk[r*16];
          imma(acc[r&3], w.x&m, w.y&m, w.z&m, w.w&m, b.x, b.y); }
      }
      cb += nch;
    } else if (MODE == 2) {
      // all chunks of this warp in the piece at once: load weights + B fragments first
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece);
      for (int c = first; c < nch; c += 2*W) {
        const bool two = c + W < nch;
        uint4 w0 = pc[c*32+lane]; uint4 w1 = two ? pc[(c+W)*32+lane] : make_uint4(0,0,0,0);
        uint2 b0[8], b1[8];
#pragma unroll
        for (int r=0;r<8;++r){ b0[r] = make_uint2(0,0); b1[r] = make_uint2(0,0);
          if (lane<16) { b0[r] = ((const uint2*)xf)[((c*8+r)&31)*16+lane]; if (two) b1[r] = ((const uint2*)xf)[(((c+W)*8+r)&31)*16+lane]; } }
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r;
          imma(acc[r&3], w0.x&m, w0.y&m, w0.z&m, w0.w&m, b0[r].x, b0[r].y);
          if (two) imma(acc[(r+2)&3], w1.x&m, w1.y&m, w1.z&m, w1.w&m, b1[r].x, b1[r].y); }
      }
      cb += nch;
    } else if (MODE == 1) {
      int first = warp - cb % W; if (first < 0) first += W;
      const uint4* pc = (const uint4*)(sm + s*piece);
      for (int c = first; c < nch; c += W) {
        uint4 w = pc[c*32+lane];
#pragma unroll
        for (int r=0;r<8;++r){ uint32_t m = 0x01010101u<<r; uint2 b = make_uint2(0,0); if (lane<16) b = ((const uint2*)xf)[((c*8+r)&31)*16+lane];
          imma(acc[r&3], w.x&m, w.y&m, w.z&m, w.w&m, b.x, b.y); }
      }
      cb += nch;
    } else { x ^= ((const uint32_t*)(sm + s*piece))[threadIdx.x]; }
    __syncwarp(); if (lane==0) mbar_arrive(&empty[s]); if(++s==slots){s=0;ph^=1;}
  }
  int t = x; for (int a=0;a<4;++a) t += acc[a][0]+acc[a][1]+acc[a][2]+acc[a][3];
  for (int a=0;a<8;++a) t += acc8[a][0]+acc8[a][1]+acc8[a][2]+acc8[a][3];
  if (t == 0x7654321) out[0] = t;
}
int main(){
  size_t total = (size_t)2<<30; uint8_t* src; CK(cudaMalloc(&src, total)); CK(cudaMemset(src, 0x5a, total)); int* out; CK(cudaMalloc(&out, 64));
  int grid = 148; size_t per_cta = (total/grid) & ~(size_t)65535;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  void (*ks[6])(const uint8_t*, size_t, int, int, int*) = {ring<3,15>, ring<6,15>, ring<7,15>, ring<6,8>, ring<7,8>, ring<7,12>};
  const char* names[6] = {"lean W=15", "pred W=15", "pair W=15", "pred W=8", "pair W=8", "pair W=12"};
  int threads[6] = {512, 512, 512, 288, 288, 416};
  for (int v = 0; v < 6; ++v) {
    CK(cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, 227*1024));
    for (int piece : {8192, 16384}) for (int slots : {8, 12}) {
      size_t smem = piece*slots + 64*8 + 4096;
      if (smem > 227*1024) continue;
      ks[v]<<<grid,threads[v],smem>>>(src, per_cta, piece, slots, out); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); ks[v]<<<grid,threads[v],smem>>>(src, per_cta, piece, slots, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-11s piece=%6d slots=%2d  %7.0f GB/s\n", names[v], piece, slots, per_cta*grid/ms/1e6);
    }
  }
  return 0;
}
