// Dense int8 tensor-core rate of the instruction shape the TRSM issues: tcgen05.mma.cta_group::2
// .kind::i8 M=256 (a CTA pair on one TPC) x N x K=32, back to back from fixed shared-memory operands
// (128B swizzle, K-major) into TMEM, one commit (multicast to both CTAs) every 64 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak_pair tools/i8_peak_pair.cu
// Usage: tools/i8_peak_pair [N ...]   (default 224 256)
//        tools/i8_peak_pair --sustain SECONDS [N [rand]]   (back to back; rand: TRSM-like data)
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    i8_peak_pair_kernel(int iters, int N, int* sink, int rnd) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned long long bar;
  __shared__ unsigned tslot;
  const unsigned IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (((unsigned)N >> 3) << 17) |
                         ((256u >> 4) << 24);
  const int warp = threadIdx.x >> 5;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  // operands: a fixed pattern (i & 3), or -- rnd -- the TRSM's data statistics: A (genotype tile,
  // first 16 KB) dosages {0,1,2}, B (slices) uniformly random int8 (toggle activity sets power)
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u + 0x9E3779B9u * (blockIdx.x + 1);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    const bool a_reg = i < 16 * 1024;   // rnd 1: A {0,1,2}, B random; rnd 2: swapped;
    //                                     rnd 3: A {0,1,2}, B random non-negative [0, 127]
    unsigned char v = (unsigned char)(i & 3);
    if (rnd == 1) v = a_reg ? (unsigned char)(h % 3) : (unsigned char)h;
    if (rnd == 2) v = a_reg ? (unsigned char)h : (unsigned char)(h % 3);
    if (rnd == 3) v = a_reg ? (unsigned char)(h % 3) : (unsigned char)(h & 127);
    smem[i] = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned tmem = tslot;
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned sa = smem_u32(smem);
      unsigned long long da = (unsigned long long)((sa >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
      unsigned long long db = da + ((16 * 1024) >> 4);
      for (int j = 0; j < 64; ++j) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da + 2 * (j & 3)), "l"(db + 2 * (j & 3)), "r"(IDESC), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(smem_u32(&bar)), "h"((unsigned short)3));
    }
    if (threadIdx.x == 0) {
      asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)), "r"(phase));
    }
    phase ^= 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) {
    int v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (v == 12345) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
  }
}

int main(int argc, char** argv) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  const size_t smem = 48 * 1024;
  CK(cudaFuncSetAttribute(i8_peak_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = prop.multiProcessorCount & ~1;
  if (argc > 2 && std::string(argv[1]) == "--sustain") {
    // sustained rate: back-to-back launches for S seconds (the board reaches its power cap);
    // the rate over everything after the first second
    const double secs = atof(argv[2]);
    const int N = argc > 3 ? atoi(argv[3]) : 224;
    const int rnd = argc <= 4 ? 0 : std::string(argv[4]) == "rand" ? 1
                  : std::string(argv[4]) == "swap" ? 2 : std::string(argv[4]) == "pos" ? 3 : 0;
    const int iters = 2000;
    const double ops1 = 2.0 * 256 * N * 32 * 64.0 * iters * (grid / 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double total_ms = 0.0, ops = 0.0, warm_ms = 0.0;
    while (total_ms < secs * 1e3) {
      cudaEventRecord(a);
      for (int k = 0; k < 16; ++k) i8_peak_pair_kernel<<<grid, 128, smem>>>(iters, N, sink, rnd);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (total_ms >= 1000.0) {
        warm_ms += ms;
        ops += 16 * ops1;
      }
      total_ms += ms;
    }
    printf("int8 tcgen05 cta_group::2 M256 N%d K32 x %d SMs, %s operands, sustained %.1f s: "
           "%.1f TOPS\n", N, grid, rnd == 1 ? "TRSM-like random" : rnd == 2 ? "A random, B {0,1,2}" : rnd == 3 ? "B random [0,127]" : "i&3 pattern", total_ms / 1e3,
           ops / warm_ms / 1e9);
    return 0;
  }
  const int nn = argc > 1 ? argc - 1 : 2;
  for (int a = 0; a < nn; ++a) {
    const int N = argc > 1 ? atoi(argv[a + 1]) : (a == 0 ? 224 : 256);
    for (int rep = 0; rep < 3; ++rep) {
      const int iters = rep == 0 ? 10 : 2000;
      cudaEventRecord(e0);
      i8_peak_pair_kernel<<<grid, 128, smem>>>(iters, N, sink, 0);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 256 * N * 32 * 64.0 * iters * (grid / 2);
      if (rep) printf("int8 tcgen05 cta_group::2 M256 N%d K32 x %d SMs: %.1f TOPS (%.3f ms)\n", N,
                      grid, ops / ms / 1e9, ms);
    }
  }
  return 0;
}
