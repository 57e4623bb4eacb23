// Dense int8 tensor-core peak on this B200 (roofline denominator of the int8 TRSM):
// every CTA (one per SM) issues tcgen05.mma.cta_group::1.kind::i8 M=128 N=256 K=32 back to back
// from fixed shared-memory operands into TMEM, committing to an mbarrier every 64 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// usage: tools/i8_peak [N ...]  (MMA N per instruction, default 256: tests N granularity)
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int N, int* sink, int sw32) {
  const unsigned IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (((unsigned)N >> 3) << 17) | ((128u >> 4) << 24);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned long long bar;
  __shared__ unsigned tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) smem[i] = (unsigned char)(i & 3);
  if (threadIdx.x == 0) {
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
  if (threadIdx.x == 0) {
    const unsigned sa = smem_u32(smem);
    // sw32 (env GG_PEAK_SW32=1 on the host -> arg): the Ozaki GEMM's SWIZZLE_32B K-major operands
    // (32-byte rows, 8-row groups 256 B apart), the same descriptor for every k step
    unsigned long long da = sw32
        ? (unsigned long long)((sa >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61)
        : (unsigned long long)((sa >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    unsigned long long db = da + ((16 * 1024) >> 4);
    const int kstep = sw32 ? 0 : 2;
    unsigned phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 64; ++j) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da + kstep * (j & 3)), "l"(db + kstep * (j & 3)), "r"(IDESC), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
      asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)), "r"(phase));
      phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 0) {
    int v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (v == 12345) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
  }
}

int main(int argc, char** argv) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  const size_t smem = 48 * 1024;
  CK(cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sw32 = getenv("GG_PEAK_SW32") != nullptr;
  if (sw32) printf("# SWIZZLE_32B operands (the Ozaki GEMM's layout)\n");
  for (int a = 0; a < (argc > 1 ? argc - 1 : 1); ++a) {
    const int N = argc > 1 ? atoi(argv[a + 1]) : 256;
    for (int rep = 0; rep < 3; ++rep) {
      const int iters = rep == 0 ? 10 : 2000;
      cudaEventRecord(e0);
      i8_peak_kernel<<<prop.multiProcessorCount, 128, smem>>>(iters, N, sink, sw32);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 128 * N * 32 * 64.0 * iters * prop.multiProcessorCount;
      printf("int8 tcgen05 M128 N%d K32 x %d SMs: %.1f TOPS (%.3f ms)\n", N,
             prop.multiProcessorCount, ops / ms / 1e9, ms);
    }
  }
  return 0;
}
