// Can integer (64-bit Shoup, fma/alu pipes) butterflies run beside FP64
// butterflies (FP64 pipe) on one SM and add throughput?  Each warp runs one
// kind; `int_every` selects which warps take the integer form.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_bfly tools/mix_bfly.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;

__device__ __forceinline__ void fp_bfly(double& x, double& y, double w, double wq, double q) {
  const double M = 6755399441055744.0;
  const double h = y * w;
  const double k = __fma_rn(y, wq, M) - M;
  const double l = __fma_rn(y, w, -h);
  const double r = __fma_rn(-k, q, h) + l;
  const double a = x;
  x = a + r;
  y = a - r;
}
__device__ __forceinline__ void int_bfly(uint64_t& u, uint64_t& v, uint64_t w, uint64_t wp, uint64_t q) {
  const uint64_t hq = __umul64hi(v, wp);
  const uint64_t t = v * w - hq * q;
  const uint64_t uu = u >= 2 * q ? u - 2 * q : u;
  u = uu + t;
  v = uu - t + 2 * q;
}

__global__ void k_mix(uint64_t* out, int int_every, uint64_t qi, uint64_t w, uint64_t wp, double q, double wd,
                      double wq) {
  const int warp = threadIdx.x / 32;
  uint64_t s = 0;
  if (int_every > 0 && warp % int_every == int_every - 1) {
    uint64_t u[CH], v[CH];
    for (int c = 0; c < CH; c++) { u[c] = threadIdx.x * 7 + c; v[c] = blockIdx.x * 13 + c; }
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int c = 0; c < CH; c += 2) int_bfly(u[c], u[c + 1], w, wp, qi), int_bfly(v[c], v[c + 1], w, wp, qi);
    }
    for (int c = 0; c < CH; c++) s ^= u[c] ^ v[c];
  } else {
    double x[CH], y[CH];
    for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 7 + c; y[c] = blockIdx.x * 13 + c; }
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int c = 0; c < CH; c += 2) fp_bfly(x[c], x[c + 1], wd, wq, q), fp_bfly(y[c], y[c + 1], wd, wq, q);
      // keep the values bounded: centred reduction every 2 iterations
      if (it & 1) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
          const double M = 6755399441055744.0;
          const double k = __fma_rn(x[c], 1.0 / q, M) - M;
          x[c] = __fma_rn(-k, q, x[c]);
          const double k2 = __fma_rn(y[c], 1.0 / q, M) - M;
          y[c] = __fma_rn(-k2, q, y[c]);
        }
      }
    }
    for (int c = 0; c < CH; c++) s ^= (uint64_t)__double_as_longlong(x[c] + y[c]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int threads = 256;
  uint64_t* out;
  cudaMalloc(&out, (size_t)p.multiProcessorCount * 16 * threads * 8);
  uint64_t q = 1125899903827969ull, w = 123456789012345ull;
  uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8}) {
    const int blocks = p.multiProcessorCount * bps;
    for (int ie : {0, 1, 2, 3, 4, 6, 8}) {
      k_mix<<<blocks, threads>>>(out, ie, q, w, wp, (double)q, (double)w, (double)w / (double)q);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; r++)
        k_mix<<<blocks, threads>>>(out, ie, q, w, wp, (double)q, (double)w, (double)w / (double)q);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bfly = (double)blocks * threads * ITERS * CH * 5;   // butterflies (CH values = CH bflys per iter)
      printf("CTAs/SM %d  int warps 1/%d: %8.3f ms  %8.1f G butterflies/s\n", bps, ie, ms / 5, bfly / (ms * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
