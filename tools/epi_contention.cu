// Does FP64 / conversion / integer arithmetic in epilogue warps slow down while the same SM's
// tensor core runs tcgen05.mma.kind::i8 back to back?  Prints cycles per dependent step and per
// independent instruction, with and without a concurrent MMA stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/epi_contention tools/epi_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
constexpr unsigned IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
constexpr int STEPS = 512;

__global__ void __launch_bounds__(192, 1) k(int mma_on, long long* out, double seed) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned long long bar;
  __shared__ unsigned tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) smem[i] = (unsigned char)(i & 3);
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned tmem = tslot;
  if (warp == 0) {
    if (lane == 0 && mma_on) {
      const unsigned sa = smem_u32(smem);
      unsigned long long da = (unsigned long long)((sa >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
      unsigned long long db = da + ((16 * 1024) >> 4);
      unsigned phase = 0;
      while (!stop) {
        for (int j = 0; j < 16; ++j)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(da + 2 * (j & 3)), "l"(db + 2 * (j & 3)), "r"(IDESC), "r"(1));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)), "r"(phase));
        phase ^= 1;
      }
    }
  } else if (warp >= 2) {
    // let the MMA stream start
    long long t0 = clock64();
    while (clock64() - t0 < 20000) {}
    double x = seed + threadIdx.x, y = 1.0000001, z = 0.9999999;
    long long r[8];
    // 1: dependent DFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS; ++i) { x = fma(x, y, z); }
    r[0] = clock64() - t0;
    // 2: 8 independent DFMA chains
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS / 8; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = fma(a0, y, z); a1 = fma(a1, y, z); a2 = fma(a2, y, z); a3 = fma(a3, y, z);
        a4 = fma(a4, y, z); a5 = fma(a5, y, z); a6 = fma(a6, y, z); a7 = fma(a7, y, z);
      }
    }
    r[1] = clock64() - t0;   // 8 * STEPS instructions
    // 3: int -> double conversions, independent
    int iv = (int)x;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS / 4; ++i) {
      c0 += (double)(iv + i); c1 += (double)(iv - i); c2 += (double)(iv ^ i); c3 += (double)(iv | i);
    }
    r[2] = clock64() - t0;   // STEPS cvts + STEPS dadds (4 chains)
    // 4: dependent FP32 FMA chain
    float f = (float)x, fy = 1.0000001f, fz = 0.9999999f;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS; ++i) { f = fmaf(f, fy, fz); }
    r[3] = clock64() - t0;
    // 5: dependent int32 IMAD chain
    unsigned u = (unsigned)iv;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS; ++i) { u = u * 2654435761u + 12345u; }
    r[4] = clock64() - t0;
    // 6: dependent DADD chain
    double d = x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < STEPS; ++i) { d = d + z; }
    r[5] = clock64() - t0;
    if (threadIdx.x == 64 && blockIdx.x == 0) {
      for (int j = 0; j < 6; ++j) out[mma_on * 8 + j] = r[j];
    }
    if (x + a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + c0 + c1 + c2 + c3 + f + u + d == 1.2345) out[15] = 1;
    __syncwarp();
    asm volatile("bar.sync 1, 128;\n");
    if (threadIdx.x == 64) stop = 1;
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 16 * 8);
  cudaMemset(out, 0, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int rep = 0; rep < 2; ++rep)
    for (int on = 0; on < 2; ++on) k<<<148, 192, 48 * 1024>>>(on, out, 1.0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA %s\n", cudaGetErrorString(e)); return 1; }
  long long h[16];
  cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
  const char* names[6] = {"DFMA dependent (cyc/step)", "DFMA 8 indep (cyc/instr)", "I2F.F64+DADD 4 chains (cyc/cvt)",
                          "FFMA dependent (cyc/step)", "IMAD dependent (cyc/step)", "DADD dependent (cyc/step)"};
  const double div[6] = {STEPS, 8.0 * STEPS, STEPS, STEPS, STEPS, STEPS};
  for (int j = 0; j < 6; ++j)
    printf("%-34s  no MMA %7.2f   with MMA %7.2f\n", names[j], h[j] / div[j], h[8 + j] / div[j]);
  return 0;
}
