// Integer / FP64 modular-arithmetic throughput microbenchmark for B200 (sm_100a).
// Measures the instruction mixes the RNS-CKKS kernels are built from, so the
// ALU roofline in DESIGN.md is a measured number, not a guess.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peak_int tools/peak_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

// 64-bit Shoup butterfly: U' = U + W*V mod q (lazy [0,2q)), V' = U - W*V + 2q
__global__ void k_shoup_bfly(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp) {
  uint64_t u[CH], v[CH];
  for (int c = 0; c < CH; c++) { u[c] = threadIdx.x * 7 + c; v[c] = blockIdx.x * 13 + c; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint64_t hq = __umul64hi(v[c], wp);
      uint64_t t = v[c] * w - hq * q;
      uint64_t uu = u[c] >= 2 * q ? u[c] - 2 * q : u[c];
      u[c] = uu + t;
      v[c] = uu - t + 2 * q;
    }
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; c++) s ^= u[c] ^ v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// full 64x64->128 MAC into 128-bit accumulator
__global__ void k_mac128(uint64_t* out, const uint64_t* __restrict__ bvals) {
  uint64_t lo[CH], hi[CH], a[CH];
  for (int c = 0; c < CH; c++) { lo[c] = 0; hi[c] = 0; a[c] = (threadIdx.x * 977 + c) | (1ull << 49); }
  uint64_t b = bvals[threadIdx.x & 31];
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint64_t pl = a[c] * b, ph = __umul64hi(a[c], b);
      asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo[c]), "+l"(hi[c]) : "l"(pl), "l"(ph));
      a[c] += pl >> 60;
    }
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; c++) s ^= lo[c] ^ hi[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 25-bit split MAC: 4 IMAD.WIDE.U32 into three 64-bit accumulators
__global__ void k_mac_split(uint64_t* out, const uint64_t* __restrict__ bvals) {
  uint64_t c0[CH], c1[CH], c2[CH];
  uint32_t a0[CH], a1[CH];
  for (int c = 0; c < CH; c++) { c0[c] = c1[c] = c2[c] = 0; a0[c] = threadIdx.x * 31 + c; a1[c] = c * 7 + 1; }
  uint64_t bb = bvals[threadIdx.x & 31];
  uint32_t b0 = (uint32_t)bb & 0x1ffffff, b1 = (uint32_t)(bb >> 25);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      c0[c] += (uint64_t)a0[c] * b0;
      c1[c] += (uint64_t)a0[c] * b1;
      c1[c] += (uint64_t)a1[c] * b0;
      c2[c] += (uint64_t)a1[c] * b1;
      a0[c] ^= (uint32_t)c0[c] & 7;
    }
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; c++) s ^= c0[c] ^ c1[c] ^ c2[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out) {
  double x[CH];
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-3 + c;
  double m = 0.999999, a = 1e-7;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fma(x[c], m, a);
  }
  double s = 0;
  for (int c = 0; c < CH; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 Shoup-style modmul by constant w (q < 2^50): r = a*w mod q via exact fma error
__global__ void k_fp64_modmul(double* out, double q, double w, double wq) {
  double x[CH];
  for (int c = 0; c < CH; c++) x[c] = (double)(threadIdx.x * 1009 + c);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      double hi = x[c] * w;
      double lo = fma(x[c], w, -hi);
      double qt = rint(x[c] * wq);
      double r = fma(-qt, q, hi) + lo;
      r = r < 0 ? r + q : r;
      x[c] = r;
    }
  }
  double s = 0;
  for (int c = 0; c < CH; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_copy(const ulonglong2* __restrict__ a, ulonglong2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d MB clock %d MHz\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, clk / 1000);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  size_t nth = (size_t)blocks * threads;
  uint64_t* out; CK(cudaMalloc(&out, nth * 8));
  uint64_t* bv; CK(cudaMalloc(&bv, 32 * 8));
  uint64_t hb[32]; for (int i = 0; i < 32; i++) hb[i] = 0x3ffffffffffffull - i * 12345;
  CK(cudaMemcpy(bv, hb, sizeof(hb), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint64_t q = 1125899903827969ull, w = 123456789012345ull;
  uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  double ops = (double)nth * ITERS * CH;
  auto run = [&](const char* name, auto launch, double per) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double rate = ops * 5 / (ms * 1e-3);
    printf("%-14s %8.3f ms  %10.2f G ops/s  (%.1f G %s/s)\n", name, ms / 5, rate / 1e9, rate * per / 1e9, "units");
  };
  run("shoup_bfly", [&] { k_shoup_bfly<<<blocks, threads>>>(out, q, w, wp); }, 1.0);
  run("mac128", [&] { k_mac128<<<blocks, threads>>>(out, bv); }, 1.0);
  run("mac_split25", [&] { k_mac_split<<<blocks, threads>>>(out, bv); }, 1.0);
  run("dfma", [&] { k_dfma<<<blocks, threads>>>((double*)out); }, 1.0);
  run("fp64_modmul", [&] { k_fp64_modmul<<<blocks, threads>>>((double*)out, (double)q, (double)w, (double)w / (double)q); }, 1.0);
  CK(cudaGetLastError());
  // HBM copy bandwidth (read+write bytes)
  size_t nbytes = (size_t)4 << 30;
  void *a, *b; CK(cudaMalloc(&a, nbytes)); CK(cudaMalloc(&b, nbytes));
  cudaMemset(a, 1, nbytes);
  size_t n16 = nbytes / 16;
  for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    k_copy<<<grid, 512>>>((ulonglong2*)a, (ulonglong2*)b, n16);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k_copy<<<grid, 512>>>((ulonglong2*)a, (ulonglong2*)b, n16);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid %5d: %.1f GB/s\n", grid, 2.0 * nbytes * 5 / (ms * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
