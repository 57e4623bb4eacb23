// Device side of the synthetic BASELINE generator (bench / test data only; not on the timed path).
//
// Counter-based splitmix64 streams keyed by (seed, stream, counter): the construction of the
// reference's datagen.py:35-52, so the int8 genotypes drawn here are bit-identical to the host
// generator (paper_1304_2272_b200/datagen.py) and to the reference's gen_dataset genotype stream
// (datagen.py:139-146: u1 counter j*n+i, u2 counter (m+j)*n+i, G = [u1<f] + [u2<f]).
// Arithmetic that feeds a comparison is rounded step by step (__dmul_rn/__dadd_rn) so no FMA
// contraction can change a bit.
#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr unsigned long long GOLDEN = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform_at(unsigned long long key, unsigned long long idx) {
  const unsigned long long u = mix64((idx + 1ULL) * GOLDEN + key);
  return __dmul_rn((double)(u >> 11), 1.1102230246251565e-16);   // 2^-53
}

__global__ void gen_kernel(unsigned long long key_maf, unsigned long long key_geno, int n, int np,
                           long long m, long long first, int cnt, double maf_lo, double maf_span,
                           int8_t* __restrict__ G, long long ldg, double* __restrict__ Z,
                           long long ldz) {
  const int j = blockIdx.y;
  if (j >= cnt) return;
  const long long snp = first + j;
  const double f = __dadd_rn(maf_lo, __dmul_rn(uniform_at(key_maf, (unsigned long long)snp), maf_span));
  const double two_f = __dmul_rn(2.0, f);
  const double sd = sqrt(__dmul_rn(two_f, __dsub_rn(1.0, f)));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    if (i < n) {
      const double u1 = uniform_at(key_geno, (unsigned long long)(snp * n + i));
      const double u2 = uniform_at(key_geno, (unsigned long long)((m + snp) * n + i));
      const int g = (u1 < f ? 1 : 0) + (u2 < f ? 1 : 0);
      if (G != nullptr) G[i + j * ldg] = (int8_t)g;
      if (Z != nullptr) Z[i + j * ldz] = __ddiv_rn(__dsub_rn((double)g, two_f), sd);
    } else if (Z != nullptr) {
      Z[i + j * ldz] = 0.0;
    }
  }
}

unsigned long long host_mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace

int gen_genotypes_run(unsigned long long seed, int stream_maf, int stream_geno, int n, long long m,
                      long long first, int cnt, double maf_lo, double maf_hi, int8_t* G,
                      long long ldg, double* Z, int ldz, cudaStream_t s) {
  const int np = pad_rows(n);
  if (n < 1 || cnt < 0 || first < 0 || first + cnt > m) {
    set_error("gen_genotypes: bad range");
    return GG_EARG;
  }
  if ((G != nullptr && ldg < n) || (Z != nullptr && ldz < np)) {
    set_error("gen_genotypes: leading dimension too small");
    return GG_EDIM;
  }
  if (cnt == 0) return GG_OK;
  if (cnt > 65535) {
    set_error("gen_genotypes: at most 65535 SNPs per call");
    return GG_EARG;
  }
  const unsigned long long key_maf = host_mix64(seed * GOLDEN + (unsigned long long)stream_maf);
  const unsigned long long key_geno = host_mix64(seed * GOLDEN + (unsigned long long)stream_geno);
  int gx = (np + 255) / 256;
  if (gx > 64) gx = 64;
  dim3 grid(gx, cnt);
  // maf span rounded on the host exactly like the reference: (hi - lo) first (datagen.py:125-126)
  const double span = maf_hi - maf_lo;
  gen_kernel<<<grid, 256, 0, s>>>(key_maf, key_geno, n, np, m, first, cnt, maf_lo, span, G, ldg, Z,
                                  ldz);
  GG_LAUNCH_CHECK("gen_kernel");
  return GG_OK;
}

}  // namespace gg
