// FP64 peak microbenchmarks for the roofline denominator (DFMA pipe and DMMA tensor pipe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16_kernel(double* out, int iters) {
  // m16n8k16: A 8 regs, B 4 regs, C 4 regs per thread
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.999999 - i * 1e-12;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int j = 0; j < 4; ++j) c[k][j] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d\n", prop.name, sms);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int iters = 20000;
      dfma_kernel<8><<<sms * bps, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<8><<<sms * bps, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)threads * sms * bps;
      printf("DFMA threads=%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", threads, bps, fl / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 4000;
      dmma_kernel<8><<<sms * bps, threads>>>(d, 10);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<8><<<sms * bps, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * sms * bps;
      printf("DMMA m8n8k4 threads=%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", threads, bps, fl / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256}) {
    for (int bps : {1, 2}) {
      int iters = 1000;
      dmma16_kernel<4><<<sms * bps, threads>>>(d, 10);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma16_kernel<4><<<sms * bps, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * 8 * 16 * 4 * iters * (double)(threads / 32) * sms * bps;
      printf("DMMA m16n8k16 threads=%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", threads, bps, fl / ms / 1e9, ms);
    }
  }
  // sustained: DMMA for ~3 s
  {
    int iters = 4000;
    cudaEventRecord(e0);
    int reps = 0;
    for (; reps < 200; ++reps) dmma_kernel<8><<<sms * 2, 256>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * iters * 8.0 * sms * 2 * reps;
    printf("DMMA sustained: %.2f TFLOP/s over %.1f ms\n", fl / ms / 1e9, ms);
  }
  return 0;
}
