// Streamed TRSM on the 5th-generation tensor cores: Xbar = Linv * G for int8 dosage blocks G,
// with the FP64 inverse split error-free into int8 slices (Ozaki-style splitting).
//
// Genotype dosages {0,1,2} are exact int8.  Each row i of Linv is written as
//     Linv[i,k] = 2^e_i ( [k == i] h_i + sum_{s=0..6} a_s[i,k] 2^(-7 (s+1)) ),  a_s in [-127, 127]
// (integer diagonal head |h_i| < 2^20, e_i >= e(diagonal) - 20; residual <= 2^(e_i - 50),
// zero-mean, see "inverse slicing" below), so
//     Xbar[i,j] = 2^(e_i - 49) ( h_i G[i,j] 2^49 + sum_s 2^(7 (6 - s)) C_s[i,j] ),
//     C_s = sum_k a_s[i,k] G[k,j]
// where every C_s is an EXACT int32 product (|C_s| <= 128 * 127 n < 2^31 up to n = 132,104;
// dosages <= 2 up to 8.4e6) computed by tcgen05.mma.kind::i8; the bracket is assembled as two
// exact int64 halves and rounded once, so a column's result never depends on its position.
//
// Kernel (persistent, CTA pairs with cta_group::2, one CTA per SM, 10 warps):
//   warp 0  producer: A = 128 SNPs x 128 k int8 per CTA (TMA, 128B swizzle, k >= n zero-filled),
//           B = this CTA's half of the 7 x 32 slice rows of each of the tile's two row blocks
//           (tile-packed slices), into a 4-5-stage mbarrier ring (44 KB / stage); per-tile row
//           data (e_i, h_i, XLbar/ybar rows) by bulk copies into 2 slots; pulls tiles heavy-first
//           from a global atomic counter and posts them to a per-cluster tile queue;
//   warp 1  MMA issuer (leader CTA, one lane): D_h[256 SNPs x 224] += A . B_h^T over the pair for
//           the two row blocks h = 0, 1, int32 accumulators in TMEM (columns 0 and 256);
//   warps 2-9  two epilogue groups (group h drains row block h of the tile): tcgen05.ld each
//           SNP's 7 x 32 accumulators, recombine, store the SNP's 32 Xbar rows and/or the fused
//           per-SNP partial dots against XLbar / ybar (canonical order of gls_epilogue.cu).
// Tiles = (pairs of 32-row blocks of Linv) x (256-SNP column pairs), swept in SNP groups
// (tile_coords); row block rb needs k < 32 (rb+1).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr int S = 7;                       // int8 slices of the inverse (+ a diagonal head)
constexpr int TM = 128;                    // SNPs per tile (MMA M)
constexpr int TR = 32;                     // inverse rows per tile
constexpr int TN = S * TR;                 // MMA N = 224
constexpr int TK = 128;                    // k per pipeline stage (4 MMAs of K = 32)
constexpr int A_BYTES = TM * TK;           // 16 KB
constexpr int THREADS = 10 * 32;   // producer, MMA, two epilogue groups of 4 warps
constexpr int ACC_COLS = 256;              // TMEM columns per accumulator buffer (TN used)
static_assert(S == 7, "tmem_ld_rows8 and the hi/lo recombination are written for 7 slices");
constexpr int HEAD_BITS = 20;              // e'_i >= e(diagonal) - HEAD_BITS: |h_i| < 2^20

struct I8Args {
  int N;            // SNP columns
  int num_rb;       // np / 32
  int num_nt;       // ceil(N / 128)
  double* X;        // Xbar, column-major, leading dimension ldx (nullptr: not materialised)
  long long ldx;
  const int* expo;  // slice metadata: e'_i per inverse row (np), then the heads h_i (np)
  const signed char* G;   // the dosages (for the head term h_i g_i of the diagonal)
  long long ldg;
  int n;
  // fused epilogue reductions (canonical order of gls_epilogue.cu): partial dots of each SNP's
  // 32-row block against XLbar (q columns, ld ldxl) and ybar -> P[(rb*(q+2) + k)*N + col]
  int q;
  const double* XL;
  long long ldxl;
  const double* y;
  double* P;        // nullptr: no partials
  const int* gate;  // device flag: the kernel runs only if *gate == gate_value (nullptr: always)
  int gate_value;
  int* tile_counter;  // zeroed before the launch: clusters take tiles dynamically, heavy first
  int rd_bytes;       // bytes per row-data slot (rd_bytes(q, P != nullptr))
  int grp_pp;         // 256-SNP tile pairs per SNP group (tile_coords)
  int order;          // tile order inside a group (tile_coords): 0 heavy first, 1 zigzag
  int quad_interleave;  // QUAD tiles: B-stationary MMA order (both A tiles per slice k-chunk)
  int whatif;         // measurement only (GG_I8_WHATIF bits; results invalid): 1 no genotype
                      // (A) loads, 2 no slice (B) loads, 4 no epilogue work
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// K-major, 128-byte-swizzled shared-memory matrix descriptor (rows of 128 B, 8-row groups
// 1024 B apart): start >> 4, LBO = 1, SBO = 1024 >> 4, version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ unsigned long long smem_desc(unsigned saddr) {
  return (unsigned long long)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

// 2^e as a double for |e| < 1022 (exact; built from the exponent bits, no libm call)
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// Tile t -> (row block rb, SNP tile nt).  The num_nt SNP tiles are cut into groups of grp; the
// groups are swept one after the other, and inside a group the row blocks heavy first with a row
// block's SNP tiles together (grp bounds the genotype working set that L2 has to hold while
// every row block re-reads it).
// order 1 (zigzag): inside a group the row blocks alternate heavy / light (the i-th heaviest, then
// the i-th lightest), so a short tile's epilogue overlaps a long tile's MMAs instead of a run of
// short, epilogue-bound tiles ending every group.
__device__ __forceinline__ void tile_coords(int t, int num_rb, int num_nt, int grp, int& rb,
                                            int& nt, int order = 0) {
  const int g = t / (num_rb * grp);
  const int t1 = t - g * num_rb * grp;
  const int w = min(grp, num_nt - g * grp);     // the last group may be narrower
  const int i = t1 / w;
  rb = (order == 1) ? ((i & 1) ? (i >> 1) : num_rb - 1 - (i >> 1)) : num_rb - 1 - i;
  nt = g * grp + t1 % w;
}

// ---- CTA-pair kernel (cta_group::2) ------------------------------------------------------------
// A cluster of 2 CTAs on a TPC computes 256-SNP x (S x 32)-column products with M = 256 MMAs
// issued by the leader: each CTA stages its own 128 SNPs (A) and HALF of the 224 slice rows of a
// row block (B is split along N: CTA0 slices 0-2 + rows 0-15 of slice 3, CTA1 the rest).  Both
// CTAs' TMA loads complete on the leader's "full" barrier; the leader's commits are multicast to
// both CTAs' "empty" / "accumulator full" barriers; both CTAs' epilogue threads release an
// accumulator on the leader's "accumulator empty" barrier.
constexpr int P_B_ROWS = TN / 2;                    // 112 slice rows per CTA of the pair
constexpr int P_B_BYTES = P_B_ROWS * TK;             // 14 KB
// per-row-block data staged by the producer with bulk copies: e_i and h_i (32 ints each), then
// the block's 32 rows of XLbar's q columns and of ybar (sized for the launch's q: a.rd_bytes)
constexpr int RD_COLS_OFF = 2 * TR * 4;   // e'_i, then the diagonal heads h_i
__host__ __device__ constexpr int rd_bytes(int q, bool partials) {
  return RD_COLS_OFF + (partials ? (q + 1) * TR * 8 : 0);
}
// dynamic tile queue: TQ slots, posted by the leader's producer to both CTAs
constexpr int TQ = 8;
constexpr unsigned IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(TN >> 3) << 17) |
                            ((unsigned)(2 * TM >> 4) << 24);
constexpr unsigned PEER_MASK = 0xFEFFFFFFu;          // clear the CTA-rank bit: the leader's copy

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" :::
                   "memory");
}
__device__ __forceinline__ void tma_2d_pair(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_4d_pair(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(unsigned d_tmem, unsigned long long a,
                                            unsigned long long b, unsigned accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC2), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(unsigned bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(bar),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITQ_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITQ_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// the same shared-memory offset in the other CTA of the pair
__device__ __forceinline__ unsigned mapa_peer(unsigned saddr) {
  unsigned r, peer;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  peer = r ^ 1u;
  unsigned out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(saddr), "r"(peer));
  return out;
}
__device__ __forceinline__ void st_cluster_s32(unsigned addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_release(unsigned bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// contiguous global -> own shared memory copy (row data), completing on the CTA's own barrier
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst),
      "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

// 8 rows x all S slices of one accumulator quarter: v[s][r] = C_s of row r (7 loads, one wait)
__device__ __forceinline__ void tmem_ld_rows8(unsigned taddr, int (&v)[S][8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%56];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%57];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%58];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%59];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [%60];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%40,%41,%42,%43,%44,%45,%46,%47}, [%61];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%48,%49,%50,%51,%52,%53,%54,%55}, [%62];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]), "=r"(v[0][6]), "=r"(v[0][7]),
        "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]), "=r"(v[1][6]), "=r"(v[1][7]),
        "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[2][4]), "=r"(v[2][5]), "=r"(v[2][6]), "=r"(v[2][7]),
        "=r"(v[3][0]), "=r"(v[3][1]), "=r"(v[3][2]), "=r"(v[3][3]), "=r"(v[3][4]), "=r"(v[3][5]), "=r"(v[3][6]), "=r"(v[3][7]),
        "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[4][2]), "=r"(v[4][3]), "=r"(v[4][4]), "=r"(v[4][5]), "=r"(v[4][6]), "=r"(v[4][7]),
        "=r"(v[5][0]), "=r"(v[5][1]), "=r"(v[5][2]), "=r"(v[5][3]), "=r"(v[5][4]), "=r"(v[5][5]), "=r"(v[5][6]), "=r"(v[5][7]),
        "=r"(v[6][0]), "=r"(v[6][1]), "=r"(v[6][2]), "=r"(v[6][3]), "=r"(v[6][4]), "=r"(v[6][5]), "=r"(v[6][6]), "=r"(v[6][7])
      : "r"(taddr + 0 * TR), "r"(taddr + 1 * TR), "r"(taddr + 2 * TR), "r"(taddr + 3 * TR), "r"(taddr + 4 * TR), "r"(taddr + 5 * TR), "r"(taddr + 6 * TR)
      : "memory");
}

// A tile is 256 SNPs x TWO adjacent 32-row blocks (2 rbp, 2 rbp + 1: the same
// 128-row slice tile, so the same k range): each stage's genotype tile A feeds two N = 224 MMAs
// (accumulators at TMEM columns 0 and 256), halving the A bytes per MAC (44 KB per stage for
// 2 x 3.67 M MACs per SM; one row block per tile with double-buffered accumulators moved 30 KB for
// 3.67 M and was 2.5-3% slower, burst and sustained, at n = 10^4 and 4*10^4).  The accumulators are single-buffered:
// epilogue group g drains row block 2 rbp + g and releases its half as soon as it is in
// registers, so the next tile's MMAs into that half wait only for the drain.
constexpr int D_STAGE_BYTES = A_BYTES + 2 * P_B_BYTES;   // 44 KB
// QUAD tiles (r02): ONE 32-row block x TWO 256-SNP column pairs -- each stage's slice tile B
// feeds two N = 224 MMAs with different genotype tiles A (accumulators at TMEM columns 0 and
// 256).  Same MACs and nearly the same bytes per stage (46 KB), but half the slice bytes per MAC:
// the slices are random low-order mantissa digits, whose movement and multiplication is where the
// power goes under the board's cap, while the genotypes are {0,1,2}.
constexpr int Q_STAGE_BYTES = 2 * A_BYTES + P_B_BYTES;   // 46 KB
constexpr int D_RD_SLOTS = 2;                            // row-data slots (x2 halves)
__host__ __device__ constexpr size_t d_smem_bytes(int stages, int rdb, bool quad = false) {
  return size_t(stages) * (quad ? Q_STAGE_BYTES : D_STAGE_BYTES) + size_t(D_RD_SLOTS) * 2 * rdb +
         1024 + 512;
}
constexpr int D_TQ_READERS = 2 + 2 * 8;   // leader MMA + peer producer + 8 epilogue warps per CTA

// NB dots of a SNP's 32 Xbar rows against NB consecutive 32-row vectors of the row-data slot (and
// x.x when XX) as NB (+1) independent FMA chains; every chain runs i = 0..31 in order.
template <int NB, bool XX>
__device__ __forceinline__ void dot_chains(const double (&acc)[TR], const double* xl,
                                           double (&s)[4], double& sxx) {
#pragma unroll
  for (int j = 0; j < NB; ++j) s[j] = 0.0;
#pragma unroll
  for (int i = 0; i < TR; ++i) {
#pragma unroll
    for (int j = 0; j < NB; ++j) s[j] = fma(acc[i], xl[j * TR + i], s[j]);
    if (XX) sxx = fma(acc[i], acc[i], sxx);
  }
}

template <int P_STAGES, bool QUAD>
__global__ void __launch_bounds__(THREADS, 1)
    trsm_i8_dual_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB3,
                        const __grid_constant__ CUtensorMap tmB1, I8Args a) {
  constexpr int STAGE = QUAD ? Q_STAGE_BYTES : D_STAGE_BYTES;
  constexpr int A_ST = QUAD ? 2 * A_BYTES : A_BYTES;          // genotype bytes per CTA stage
  constexpr int B_ST = QUAD ? P_B_BYTES : 2 * P_B_BYTES;      // slice bytes per CTA stage
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* rdata = smem + P_STAGES * STAGE;
  const int RD_BYTES = a.rd_bytes;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(rdata + D_RD_SLOTS * 2 * RD_BYTES);
  // barriers: full[P], empty[P], accf, acce[2], rdf[RD], rde[RD], tqf[TQ], tqe[TQ]
  int* tq = reinterpret_cast<int*>(bars + 2 * P_STAGES + 3 + 2 * D_RD_SLOTS + 2 * TQ);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tq + TQ);
  const unsigned sbase = smem_u32(smem);
  const unsigned rbase = smem_u32(rdata);
  const unsigned full0 = smem_u32(bars);
  const unsigned empty0 = smem_u32(bars + P_STAGES);
  const unsigned accf = smem_u32(bars + 2 * P_STAGES);
  const unsigned acce0 = smem_u32(bars + 2 * P_STAGES + 1);
  const unsigned rdf0 = smem_u32(bars + 2 * P_STAGES + 3);
  const unsigned rde0 = rdf0 + 8 * D_RD_SLOTS;
  const unsigned tqf0 = rde0 + 8 * D_RD_SLOTS;
  const unsigned tqe0 = tqf0 + 8 * TQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = cluster_rank();
  const bool leader = rank == 0;
  if (a.gate != nullptr && *a.gate != a.gate_value) return;   // uniform over the grid

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accf, 1);
    for (int h = 0; h < 2; ++h) mbar_init(acce0 + 8 * h, 2 * 4 * 32);   // both CTAs' group h
    for (int b = 0; b < D_RD_SLOTS; ++b) {
      mbar_init(rdf0 + 8 * b, 1);
      mbar_init(rde0 + 8 * b, 8 * 32);
    }
    for (int b = 0; b < TQ; ++b) {
      mbar_init(tqf0 + 8 * b, 1);
      mbar_init(tqe0 + 8 * b, D_TQ_READERS);   // leader's copy used
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * ACC_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const unsigned tmem_base = *tmem_slot;

  // tile = (row unit ru, column unit cu): dual -- row-block pair x 256-SNP pair; QUAD -- one row
  // block x two 256-SNP pairs.  Half h of the tile: row block rb_h, SNP tile nt_h (this CTA's)
  const int num_cu = QUAD ? (a.num_nt + 3) / 4 : (a.num_nt + 1) / 2;
  const int num_ru = QUAD ? a.num_rb : a.num_rb / 2;   // num_rb is a multiple of 4
  const int total = num_ru * num_cu;
  const bool partials = a.P != nullptr;
  const unsigned peer_tq = mapa_peer(smem_u32(tq));
  auto tile_at = [&](int r) -> int {
    const int slot = r % TQ;
    mbar_wait_acq_cluster(tqf0 + 8 * slot, (r / TQ) & 1);
    return *reinterpret_cast<volatile int*>(tq + slot);
  };
  auto tile_read = [&](int r) { mbar_arrive_cluster((tqe0 + 8 * (r % TQ)) & PEER_MASK); };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (int r = 0;; ++r) {
        int t;
        if (leader) {   // take the next tile (heavy first) and post it to both CTAs
          const int slot = r % TQ;
          mbar_wait(tqe0 + 8 * slot, ((r / TQ) & 1) ^ 1);
          t = atomicAdd(a.tile_counter, 1);
          if (t >= total) t = -1;
          tq[slot] = t;
          st_cluster_s32(peer_tq + 4 * slot, t);
          mbar_arrive(tqf0 + 8 * slot);
          mbar_arrive_remote_release(mapa_peer(tqf0 + 8 * slot));
        } else {
          t = tile_at(r);
          tile_read(r);
        }
        if (t < 0) break;
        int ru, cu;
        tile_coords(t, num_ru, num_cu, a.grp_pp, ru, cu, a.order);
        const int rb0 = QUAD ? ru : 2 * ru;        // the tile's (first) row block
        const int nk = (QUAD ? ru : 2 * ru + 1) / 4 + 1;
        constexpr int NRD = QUAD ? 1 : 2;          // row blocks (row data) per tile
        {   // row data of the tile's row block(s) (this CTA's own barrier)
          const int slot = r % D_RD_SLOTS;
          mbar_wait(rde0 + 8 * slot, ((r / D_RD_SLOTS) & 1) ^ 1);
          const unsigned rbar = rdf0 + 8 * slot;
          mbar_expect_tx(rbar, NRD * (2 * TR * 4 + (partials ? (a.q + 1) * TR * 8 : 0)));
          for (int h = 0; h < NRD; ++h) {
            const unsigned dst = rbase + (2 * slot + h) * RD_BYTES;
            const int row0 = (rb0 + h) * TR;
            bulk_g2s(dst, a.expo + row0, TR * 4, rbar);
            bulk_g2s(dst + TR * 4, a.expo + a.num_rb * TR + row0, TR * 4, rbar);
            if (partials) {
              for (int c = 0; c < a.q; ++c)
                bulk_g2s(dst + RD_COLS_OFF + c * TR * 8, a.XL + c * a.ldxl + row0, TR * 8, rbar);
              bulk_g2s(dst + RD_COLS_OFF + a.q * TR * 8, a.y + row0, TR * 8, rbar);
            }
          }
        }
        const int tile0 = (rb0 >> 2) * ((rb0 >> 2) + 1) / 2;
        for (int kt = 0; kt < nk; ++kt) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const unsigned fb = full0 + 8 * stage;
          if (leader)
            mbar_expect_tx(fb, 2 * (((a.whatif & 1) ? 0 : A_ST) + ((a.whatif & 2) ? 0 : B_ST)));
          const unsigned dA = sbase + stage * STAGE;
          const unsigned fbl = fb & PEER_MASK;
          auto loadB = [&](unsigned dst, const CUtensorMap* m, int c1, int c2) {
            if (a.whatif & 2) return;
            tma_4d_pair(dst, m, fbl, 0, c1, c2, tile0 + kt);
          };
          if (a.whatif & 1) {
            // what-if (timing only, results invalid): no genotype loads -- the A bytes' share of
            // the L2 -> SMEM stream and of DRAM (the leader expects only the B bytes)
          } else if (QUAD) {   // the CTA's two SNP tiles: 4 cu + rank and 4 cu + 2 + rank
            tma_2d_pair(dA, &tmA, fbl, kt * TK, (4 * cu + (int)rank) * TM);
            tma_2d_pair(dA + A_BYTES, &tmA, fbl, kt * TK, (4 * cu + 2 + (int)rank) * TM);
          } else {
            tma_2d_pair(dA, &tmA, fbl, kt * TK, (2 * cu + (int)rank) * TM);
          }
#pragma unroll
          for (int h = 0; h < (QUAD ? 1 : 2); ++h) {   // this CTA's 112 slice rows of rb0 + h
            const unsigned dB = dA + A_ST + h * P_B_BYTES;
            const int r0 = ((rb0 + h) & 3) * TR;
            if (rank == 0) {
              loadB(dB, &tmB3, r0, 0);
              loadB(dB + 3 * TR * TK, &tmB1, r0, 3);
            } else {
              loadB(dB, &tmB1, r0 + TR / 2, 3);
              loadB(dB + (TR / 2) * TK, &tmB3, r0, 4);
            }
          }
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      int stage = 0;
      unsigned phase = 0;
      for (int r = 0;; ++r) {
        const int t = tile_at(r);
        tile_read(r);
        if (t < 0) break;
        int ru, cu;
        tile_coords(t, num_ru, num_cu, a.grp_pp, ru, cu, a.order);
        const int rb0 = QUAD ? ru : 2 * ru;
        const int nk = (QUAD ? ru : 2 * ru + 1) / 4 + 1;
        for (int kt = 0; kt < nk; ++kt) {
          mbar_wait(full0 + 8 * stage, phase);
          fence_after();
          const unsigned sa = sbase + stage * STAGE;
          if (QUAD && a.quad_interleave) {
            // QUAD, B-stationary order: both genotype tiles against the same slice k-chunk back
            // to back, so the multipliers' B inputs (the random slice digits, where the int8
            // datapath's power goes) change every second MMA instead of every MMA
            if (kt == 0) {
#pragma unroll
              for (int h = 0; h < 2; ++h) mbar_wait(acce0 + 8 * h, (r & 1) ^ 1);
              fence_after();
            }
            const unsigned long long db = smem_desc(sa + A_ST);
            const int kk_end = (kt == nk - 1) ? (rb0 & 3) + 1 : TK / 32;
#pragma unroll
            for (int kk = 0; kk < TK / 32; ++kk)
              if (kk < kk_end) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  mma_i8_pair(tmem_base + h * ACC_COLS, smem_desc(sa + h * A_BYTES) + 2 * kk,
                              db + 2 * kk, (kt > 0 || kk > 0) ? 1u : 0u);
              }
          } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (kt == 0) {   // this half's accumulator drained by the previous tile's group h
              mbar_wait(acce0 + 8 * h, (r & 1) ^ 1);
              fence_after();
            }
            // dual: one genotype tile, the slices of row block rb0 + h; QUAD: genotype tile h,
            // the one row block's slices
            const unsigned long long da = smem_desc(sa + (QUAD ? h * A_BYTES : 0));
            const unsigned long long db = smem_desc(sa + A_ST + (QUAD ? 0 : h * P_B_BYTES));
            // the diagonal k tile: nonzero slices only for k < 32 (rb + 1)
            const int kk_end = (kt == nk - 1) ? ((rb0 + (QUAD ? 0 : h)) & 3) + 1 : TK / 32;
#pragma unroll
            for (int kk = 0; kk < TK / 32; ++kk)
              if (kk < kk_end)
                mma_i8_pair(tmem_base + h * ACC_COLS, da + 2 * kk, db + 2 * kk,
                            (kt > 0 || kk > 0) ? 1u : 0u);
          }
          }
          mma_commit_pair(empty0 + 8 * stage);
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(accf);
      }
    }
  } else {
    const int group = (warp - 2) >> 2;         // group g drains row block 2 rbp + g
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    for (int r = 0;; ++r) {
      const int t = tile_at(r);
      __syncwarp();
      if (lane == 0) tile_read(r);
      if (t < 0) break;
      int ru, cu;
      tile_coords(t, num_ru, num_cu, a.grp_pp, ru, cu, a.order);
      const int rb = QUAD ? ru : 2 * ru + group;
      const int nt = QUAD ? 4 * cu + 2 * group + (int)rank : 2 * cu + (int)rank;
      const int col_g = nt * TM + m, row0_g = rb * TR;
      int gq[TR / 4];
      {
        const signed char* gp = a.G + (long long)(col_g < a.N ? col_g : 0) * a.ldg + row0_g;
        if (col_g < a.N && row0_g + TR <= a.n) {
          const int4 w0 = *reinterpret_cast<const int4*>(gp);
          const int4 w1 = *reinterpret_cast<const int4*>(gp + 16);
          gq[0] = w0.x; gq[1] = w0.y; gq[2] = w0.z; gq[3] = w0.w;
          gq[4] = w1.x; gq[5] = w1.y; gq[6] = w1.z; gq[7] = w1.w;
        } else {
#pragma unroll
          for (int w = 0; w < TR / 4; ++w) {
            int v = 0;
            for (int b = 0; b < 4; ++b) {
              const int rr = row0_g + 4 * w + b;
              const int g = (col_g < a.N && rr < a.n) ? (int)gp[4 * w + b] : 0;
              v |= (g & 0xff) << (8 * b);
            }
            gq[w] = v;
          }
        }
      }
      mbar_wait(accf, r & 1);
      fence_after();
      const int slot = r % D_RD_SLOTS;
      const unsigned char* rd = rdata + (2 * slot + (QUAD ? 0 : group)) * RD_BYTES;
      const int* ex = reinterpret_cast<const int*>(rd);
      const double* cols = reinterpret_cast<const double*>(rd + RD_COLS_OFF);
      mbar_wait(rdf0 + 8 * slot, (r / D_RD_SLOTS) & 1);
      if (a.whatif & 4) {   // what-if: release at once, no loads / math / stores
        fence_before();
        mbar_arrive_cluster((acce0 + 8 * group) & PEER_MASK);
        mbar_arrive(rde0 + 8 * slot);
        continue;
      }
      const int* hd = reinterpret_cast<const int*>(rd + TR * 4);
      double acc[TR];
      const unsigned taddr = tmem_base + group * ACC_COLS + ((unsigned)(quarter * 32) << 16);
#pragma unroll
      for (int q4 = 0; q4 < TR / 8; ++q4) {
        int v[S][8];
        tmem_ld_rows8(taddr + q4 * 8, v);
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
          const int i = q4 * 8 + r8;
          const int g = (int)(signed char)((gq[i >> 2] >> (8 * (i & 3))) & 0xff);
          const long long hi = (long long)hd[i] * g * (1ll << 21) +
                               (((long long)v[0][r8] * 128 + v[1][r8]) * 128 + v[2][r8]);
          const long long lo = (((long long)v[3][r8] * 128 + v[4][r8]) * 128 + v[5][r8]) * 128 +
                               v[6][r8];
          const int e = ex[i];
          // (an I2F-free int64 -> double form -- bits(1.5 2^52) + x, constants folded into the
          // FMAs, bitwise equal -- measured no faster: profiles/r02_epilogue_forms_ab.log)
          acc[i] = fma((double)hi, pow2(e - 21), (double)lo * pow2(e - 49));
        }
      }
      fence_before();
      mbar_arrive_cluster((acce0 + 8 * group) & PEER_MASK);
      const int col = col_g;
      if (col < a.N) {
        if (a.X != nullptr) {
          double* dst = a.X + (long long)col * a.ldx + row0_g;
#pragma unroll
          for (int i = 0; i < TR; i += 2)
            *reinterpret_cast<double2*>(dst + i) = make_double2(acc[i], acc[i + 1]);
        }
        if (partials) {   // canonical order: one FMA chain over the 32 rows per dot
          // value-major partials: a warp's 32 consecutive SNPs store 256 contiguous bytes per dot
          const long long N = a.N;
          double* ppo = a.P + (long long)rb * (a.q + 2) * N + col;
          if (a.whatif & (8 | 32)) {
            // the r01 form: one dot after the other (32 | A/B knob GG_I8_EPI=2), and what-if 8
            // (timing only): only the intercept's dot and x.x, x.y stay in FP64
            const int qd = (a.whatif & 8) ? (a.q < 1 ? a.q : 1) : a.q;
            for (int k = 0; k < qd; ++k) {
              const double* xl = cols + k * TR;
              double sum = 0.0;
#pragma unroll
              for (int i = 0; i < TR; ++i) sum = fma(acc[i], xl[i], sum);
              ppo[k * N] = sum;
            }
            const double* yv = cols + a.q * TR;
            double sxx = 0.0, sxy = 0.0;
#pragma unroll
            for (int i = 0; i < TR; ++i) {
              sxx = fma(acc[i], acc[i], sxx);
              sxy = fma(acc[i], yv[i], sxy);
            }
            ppo[a.q * N] = sxx;
            ppo[(a.q + 1) * N] = sxy;
          } else {
            // the q + 1 dots against [XLbar | ybar] (ybar is vector q of the slot) and x.x as
            // independent FMA chains, four vectors at a time: each chain keeps its canonical
            // order (same bits), but a dependent DFMA takes ~158 cycles beside tcgen05 and
            // independent ones issue every ~16 -- one chain at a time left the FP64 pipe idle
            const int nv = a.q + 1;
            double sxx = 0.0;
            {
              double s4[4];
              const int c4 = nv < 4 ? nv : 4;
              if (c4 == 4) dot_chains<4, true>(acc, cols, s4, sxx);
              else if (c4 == 3) dot_chains<3, true>(acc, cols, s4, sxx);
              else if (c4 == 2) dot_chains<2, true>(acc, cols, s4, sxx);
              else dot_chains<1, true>(acc, cols, s4, sxx);
              for (int j = 0; j < c4; ++j) ppo[(long long)(j < a.q ? j : a.q + 1) * N] = s4[j];
              ppo[(long long)a.q * N] = sxx;
            }
            for (int v0 = 4; v0 < nv; v0 += 4) {
              double s4[4], unused = 0.0;
              const int c4 = nv - v0 < 4 ? nv - v0 : 4;
              const double* xl = cols + v0 * TR;
              if (c4 == 4) dot_chains<4, false>(acc, xl, s4, unused);
              else if (c4 == 3) dot_chains<3, false>(acc, xl, s4, unused);
              else if (c4 == 2) dot_chains<2, false>(acc, xl, s4, unused);
              else dot_chains<1, false>(acc, xl, s4, unused);
              for (int j = 0; j < c4; ++j) {
                const int v = v0 + j;
                ppo[(long long)(v < a.q ? v : a.q + 1) * N] = s4[j];
              }
            }
          }
        }
      }
      mbar_arrive(rde0 + 8 * slot);   // row data slot free
    }
  }
  fence_before();
  cluster_sync();   // every MMA retired and every remote arrival delivered before freeing TMEM
  fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                 "r"(2 * ACC_COLS)
                 : "memory");
  }
}

// ---- inverse slicing ---------------------------------------------------------------------------
// Row i of the inverse is split as
//     Linv[i,k] = 2^e'_i ( [k == i] h_i + sum_{s=0..6} a_s[i,k] 2^(-7 (s+1)) ),  a_s in [-127, 127]
// with e'_i = max(e_off_i, e_diag_i - HEAD_BITS) (|Linv[i,k]| < 2^e_off_i for k < i): the large
// diagonal element gets an integer head h_i (|h_i| < 2^20, applied in the epilogue as h_i g_i),
// everything else 7 slices: slices 0-5 floor (exact remainders in [0, 1): slices 1-5 and the
// last are non-negative, only slice 0 carries the sign), the last rounds to nearest,
// so the residual is zero-mean and <= 2^(e'_i - 50) (2^(e'_i - 49) in the rare clipped case):
// 50 bits below the row's largest off-diagonal entry, >= 54 below the row maximum when the
// diagonal dominates it 16x (kinship covariances: ~36x).  Measured on a kinship inverse at
// n = 1500: X errors 1.9e-15 of the column maximum (FP64 GEMM: 5.6e-16; all-truncated slices
// 5.2e-15, 6 slices 2.7e-13 -- hence 7).
// Slices are stored tile-packed: the lower triangle of 128 x 128 tiles (row tile mt, k tile kt,
// kt <= mt) at tile index mt (mt+1)/2 + kt, each tile [slice 7][row 128][k 128] int8 (112 KB):
// 3.5 np^2 + O(np) bytes (79 GB at n = 1.5e5, where a square layout would not fit a GPU).
// Metadata ("expo" in the C-ABI): e'_i (np ints) then h_i (np ints).
constexpr int ST = 128;                                  // slice tile edge
constexpr long long ST_BYTES = (long long)S * ST * ST;   // 112 KB

__host__ __device__ inline long long slice_tiles(int np) {
  const long long nt = np / ST;
  return nt * (nt + 1) / 2;
}
__device__ __forceinline__ long long slice_offset(int i, int k, int s) {   // k <= diag tile end
  const long long mt = i / ST, kt = k / ST;
  return (mt * (mt + 1) / 2 + kt) * ST_BYTES + (long long)s * ST * ST + (long long)(i % ST) * ST +
         (k % ST);
}

// Element sources for the slicing kernels: row-major square inverse, packed FP64 inverse
// (trsm_tma.cu layout), and one rank's share of a 2D block-cyclic inverse (0 where not owned).
struct SrcRowMajor {
  const double* A;
  long long ld;
  __device__ double operator()(int i, int k) const { return A[(long long)i * ld + k]; }
};
struct SrcPacked {
  const double* P;
  __device__ double operator()(int i, int k) const {
    const long long mt = i / 128;
    return P[(4 * mt * (mt + 1) + k / 16) * 2048 + (i % 128) * 16 + (k % 16)];
  }
};
struct SrcBlockCyclic {
  const double* B;
  long long ldl;
  int nb, gr, gc, pr, pc;
  __device__ double operator()(int i, int k) const {
    const int I = i / nb, J = k / nb;
    if (I % gr != pr || J % gc != pc) return 0.0;
    const long long li = (long long)(I / gr) * nb + i % nb, lk = (long long)(J / gc) * nb + k % nb;
    return B[li + lk * ldl];
  }
};

__device__ __forceinline__ int exp_of(double mx) {   // |x| < 2^e, INT_MIN for 0
  int e = INT_MIN;
  if (mx > 0.0) frexp(mx, &e);
  return e;
}

// Row exponents over what this source holds: out[i] = e_off_i (k < i), out[np + i] = e_diag_i
// (INT_MIN where absent: the distributed form MAX-reduces them over ranks).  One CTA per row.
template <class Src>
__global__ void row_exponent_kernel(int np, Src src, int* __restrict__ out) {
  const int i = blockIdx.x;
  __shared__ double red[32];
  double mx = 0.0;
  for (int k = threadIdx.x; k < i && k < np; k += blockDim.x) mx = fmax(mx, fabs(src(i, k)));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) mx = fmax(mx, red[w]);
    out[i] = exp_of(mx);
    out[np + i] = exp_of(fabs(src(i, i)));
  }
}

// meta[i] = e'_i = max(e_off, e_diag - HEAD_BITS) from [e_off | e_diag]; meta[np + i] = 0 (the
// heads are written by the slicing kernel).  In place is allowed.
__global__ void slice_meta_kernel(int np, const int* ex2, int* meta) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const int eo = ex2[i], ed = ex2[np + i];
    int e = ed == INT_MIN ? eo : (eo == INT_MIN ? ed - HEAD_BITS : max(eo, ed - HEAD_BITS));
    if (e == INT_MIN) e = 0;   // all-zero row (not an inverse row; keeps the arithmetic finite)
    meta[i] = e;
    meta[np + i] = 0;
  }
}

// Slices of row i for k < (i/128 + 1) * 128 (zero above the diagonal) given e'_i; the diagonal
// splits into the head h_i (written to meta[np + i] by the thread that sees a nonzero Linv_ii)
// and its fractional part, sliced like the other entries.  v in (-1, 1); every step is exact.
template <class Src>
__global__ void slice_rows_kernel(int np, Src src, int* __restrict__ meta,
                                  signed char* __restrict__ Sl) {
  const int i = blockIdx.x;
  const int e = meta[i];
  const int kend = (i / ST + 1) * ST;
  for (int k = threadIdx.x; k < kend; k += blockDim.x) {
    double v = (k <= i) ? src(i, k) : 0.0;
    v = (v != 0.0) ? ldexp(v, -e) : 0.0;
    if (k == i) {
      const double h = trunc(v);
      if (v != 0.0) meta[np + i] = (int)h;
      v -= h;
    }
    // truncated digits (exact remainders, |v| < 1); the last rounds to nearest instead (|q| <= 127
    // kept): a zero-mean residual of at most half a unit, which does not build up along k.  The
    // value they represent, V = sum_s c_s 128^(6-s) (|V| < 2^49, exact in int64), is then
    // re-encoded with FLOOR digits -- d_0 = floor(V / 2^42) in [-128, 127], d_1..6 the base-128
    // digits of V - d_0 2^42 in [0, 127] -- the same value, but only slice 0 carries the sign: the
    // int8 datapath's power follows the operand bits, and the sign extension of random-sign
    // digits costs ~5% of clock under the power cap (r02, profiles/r02_whatif_operands2.log).
    // (Floor digits taken directly from v are not exact: a tiny negative v leaves a remainder
    // that rounds to 1.0.)
    long long V = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double t = v * 128.0;                     // exact
      const double q = (s < S - 1) ? trunc(t) : fmin(fmax(rint(t), -127.0), 127.0);
      V = V * 128 + (long long)q;
      v = t - q;
    }
    Sl[slice_offset(i, k, 0)] = (signed char)(V >> (7 * (S - 1)));   // arithmetic: floor
#pragma unroll
    for (int s = 1; s < S; ++s)
      Sl[slice_offset(i, k, s)] = (signed char)((V >> (7 * (S - 1 - s))) & 127);
  }
}

// FP64 dosages -> int8 (exactness check: integers with |v| <= gmax); rows n .. min(ldg, n16)-1
// of each column (n16 = n rounded up to 16) are written as zero.  One warp converts a 512-row
// segment of a column: lane l takes rows 2 (32 h + l) + {0, 1}, h = 0..7, so every load
// instruction reads 512 contiguous bytes (8 in flight per thread, streaming: the dosages are read
// once and must not evict the TRSM's operands from L2) and every store writes 64 contiguous
// bytes.  HBM-bound: 8 B read + 1 B written per dosage.
__global__ void narrow_kernel(int n, int cnt, const double* __restrict__ X, long long ldx,
                              signed char* __restrict__ G, long long ldg, double gmax,
                              int* __restrict__ bad, int* __restrict__ colbad) {
  const long long nw_rows = (long long)((n + 15) & ~15) < ldg ? (long long)((n + 15) & ~15) : ldg;
  const int rows = (int)nw_rows;
  const int segs = (rows + 511) / 512;
  const long long total = (long long)segs * cnt;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const bool vec = ((ldx & 1) == 0) && ((ldg & 1) == 0) &&
                   ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(G) & 1) == 0);
  int local_bad = 0;
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; e < total;
       e += nwarps) {
    const long long j = e / segs;
    const int r0 = (int)(e - j * segs) * 512;
    const double* col = X + j * ldx + r0;
    signed char* dst = G + j * ldg + r0;
    int seg_bad = 0;
    if (vec && r0 + 512 <= n) {
      double2 v[8];
#pragma unroll
      for (int h = 0; h < 8; ++h)
        v[h] = __ldcs(reinterpret_cast<const double2*>(col) + 32 * h + lane);
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const bool ok0 = (v[h].x == trunc(v[h].x)) && fabs(v[h].x) <= gmax;
        const bool ok1 = (v[h].y == trunc(v[h].y)) && fabs(v[h].y) <= gmax;
        seg_bad |= (ok0 && ok1) ? 0 : 1;
        const unsigned w = ((unsigned)(ok0 ? (int)v[h].x : 0) & 0xffu) |
                           (((unsigned)(ok1 ? (int)v[h].y : 0) & 0xffu) << 8);
        *reinterpret_cast<unsigned short*>(dst + 2 * (32 * h + lane)) = (unsigned short)w;
      }
    } else {
#pragma unroll 1
      for (int h = 0; h < 8; ++h) {
        for (int u = 0; u < 2; ++u) {
          const int r = 2 * (32 * h + lane) + u;
          if (r0 + r >= rows) continue;
          int g = 0;
          if (r0 + r < n) {
            const double v = col[r];
            const bool ok = (v == trunc(v)) && fabs(v) <= gmax;
            seg_bad |= ok ? 0 : 1;
            g = ok ? (int)v : 0;
          }
          dst[r] = (signed char)g;
        }
      }
    }
    // the segment's column is flagged on its own: every column takes its path from its own
    // values only (a column's result never depends on its neighbours)
    if (__any_sync(0xffffffffu, seg_bad != 0)) {
      local_bad = 1;
      if (lane == 0 && colbad != nullptr) atomicOr(colbad + j, 1);
    }
  }
  if (local_bad && lane == 0) atomicOr(bad, 1);
}

// int8 dosages: per column, colbad[j] |= 1 (and *bad |= 1) if any |g| exceeds gmax (the
// exact-int32 bound for this n).  One warp per column at a time.
__global__ void range_i8_kernel(int n, int cnt, const signed char* __restrict__ G, long long ldg,
                                int gmax, int* __restrict__ bad, int* __restrict__ colbad) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  bool any = false;
  for (long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; j < cnt;
       j += nwarps) {
    bool b = false;
    for (int i = lane; i < n; i += 32) {
      const int g = G[j * ldg + i];
      b |= (g > gmax) || (g < -gmax);
    }
    if (__any_sync(0xffffffffu, b)) {
      any = true;
      if (lane == 0 && colbad != nullptr) atomicOr(colbad + j, 1);
    }
  }
  if (any && lane == 0) atomicOr(bad, 1);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_i8() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode(CUtensorMap* map, int rank, const void* base, const cuuint64_t* dims,
           const cuuint64_t* strides, const cuuint32_t* box) {
  auto fn = encode_fn_i8();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return GG_ECUDA;
  }
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (int8) failed (code " + std::to_string((int)r) + ")");
    return GG_ECUDA;
  }
  return GG_OK;
}

int sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int smem_optin() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return n;
}

}  // namespace

int i8_slices() { return S; }

size_t inverse_slices_bytes(int n) { return (size_t)slice_tiles(pad_rows(n)) * ST_BYTES; }
size_t slice_meta_ints(int n) { return 2 * (size_t)pad_rows(n); }

template <class Src>
static int slice_from(int n, Src src, signed char* Sl, int* meta, cudaStream_t s) {
  const int np = pad_rows(n);
  row_exponent_kernel<<<np, 256, 0, s>>>(np, src, meta);   // [e_off | e_diag] in place
  GG_LAUNCH_CHECK("row_exponent_kernel");
  slice_meta_kernel<<<(np + 255) / 256, 256, 0, s>>>(np, meta, meta);
  GG_LAUNCH_CHECK("slice_meta_kernel");
  slice_rows_kernel<<<np, 256, 0, s>>>(np, src, meta, Sl);
  GG_LAUNCH_CHECK("slice_rows_kernel");
  return GG_OK;
}

int slice_inverse_run(int n, const double* LinvT, int ldp, signed char* Sl, int* meta,
                      cudaStream_t s) {
  if (ldp < pad_rows(n)) {
    set_error("slice_inverse: ld must be >= gg_pad(n)");
    return GG_EDIM;
  }
  return slice_from(n, SrcRowMajor{LinvT, ldp}, Sl, meta, s);
}

int slice_packed_run(int n, const double* LinvP, signed char* Sl, int* meta, cudaStream_t s) {
  return slice_from(n, SrcPacked{LinvP}, Sl, meta, s);
}

int row_exponents_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                         int* ex2, cudaStream_t s) {
  if (nb < 1 || gr < 1 || gc < 1 || pr < 0 || pr >= gr || pc < 0 || pc >= gc) {
    set_error("row_exponents_blockcyclic: bad grid");
    return GG_EARG;
  }
  const int np = pad_rows(n);
  SrcBlockCyclic src{B, ldl, nb, gr, gc, pr, pc};
  row_exponent_kernel<<<np, 256, 0, s>>>(np, src, ex2);
  GG_LAUNCH_CHECK("row_exponent_kernel");
  return GG_OK;
}

int slice_meta_run(int n, const int* ex2, int* meta, cudaStream_t s) {
  const int np = pad_rows(n);
  slice_meta_kernel<<<(np + 255) / 256, 256, 0, s>>>(np, ex2, meta);
  GG_LAUNCH_CHECK("slice_meta_kernel");
  return GG_OK;
}

int slice_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                 int* meta, signed char* Sl, cudaStream_t s) {
  if (nb < 1 || gr < 1 || gc < 1 || pr < 0 || pr >= gr || pc < 0 || pc >= gc) {
    set_error("slice_blockcyclic: bad grid");
    return GG_EARG;
  }
  const int np = pad_rows(n);
  SrcBlockCyclic src{B, ldl, nb, gr, gc, pr, pc};
  slice_rows_kernel<<<np, 256, 0, s>>>(np, src, meta, Sl);
  GG_LAUNCH_CHECK("slice_rows_kernel");
  return GG_OK;
}

// Largest |dosage| for which every slice product 127 |g| n stays below 2^31 (exact int32).
int i8_value_bound(int n) {
  if (n < 1) return 127;
  const long long b = 2147483647LL / (128LL * (long long)n);   // slice digits in [-128, 127]
  return b >= 127 ? 127 : (int)b;
}

int range_i8_run(int n, int cnt, const signed char* G, long long ldg, int* bad, int* colbad,
                 cudaStream_t s) {
  if (cnt <= 0 || i8_value_bound(n) >= 127) return GG_OK;
  long long grid = ((long long)cnt + 7) / 8;   // 8 warps (columns) per block
  if (grid > 148LL * 16) grid = 148LL * 16;
  range_i8_kernel<<<(int)grid, 256, 0, s>>>(n, cnt, G, ldg, i8_value_bound(n), bad, colbad);
  GG_LAUNCH_CHECK("range_i8_kernel");
  return GG_OK;
}

int narrow_run(int n, int cnt, const double* X, long long ldx, signed char* G, long long ldg,
               int* bad, int* colbad, cudaStream_t s) {
  if (ldx < n || ldg < n) {
    set_error("narrow: leading dimensions too small");
    return GG_EDIM;
  }
  if (cnt <= 0) return GG_OK;
  long long grid = ((long long)((n + 511) / 512) * cnt + 7) / 8;   // 8 warps per block
  if (grid > 148LL * 16) grid = 148LL * 16;
  narrow_kernel<<<(int)grid, 256, 0, s>>>(n, cnt, X, ldx, G, ldg, (double)i8_value_bound(n), bad,
                                          colbad);
  GG_LAUNCH_CHECK("narrow_kernel");
  return GG_OK;
}

int trsm_i8_run(int n, int nrhs, const signed char* Sl, const int* expo, const signed char* G,
                long long ldg, double* X, int ldx, int* counter, cudaStream_t s) {
  return trsm_i8_fused_run(n, nrhs, Sl, expo, G, ldg, X, ldx, 0, nullptr, 0, nullptr, nullptr,
                           nullptr, 0, counter, s);
}

int trsm_i8_fused_run(int n, int nrhs, const signed char* Sl, const int* expo,
                      const signed char* G, long long ldg, double* X, int ldx, int q,
                      const double* XL, int ldxl, const double* y, double* P, const int* gate,
                      int gate_value, int* counter, cudaStream_t s) {
  const int np = pad_rows(n);
  if ((X != nullptr && ldx < np) || ldg < n || (ldg % 16) != 0 || (P != nullptr && ldxl < np)) {
    set_error("trsm_i8: ldx >= gg_pad(n), ldg >= n and ldg a multiple of 16 required");
    return GG_EDIM;
  }
  if (nrhs <= 0) return GG_OK;
  if (counter == nullptr) {
    set_error("trsm_i8: no tile counter (workspace) given");
    return GG_EARG;
  }
  if ((reinterpret_cast<uintptr_t>(Sl) | reinterpret_cast<uintptr_t>(G) |
       reinterpret_cast<uintptr_t>(X)) & 15) {
    set_error("trsm_i8: operands must be 16-byte aligned");
    return GG_EARG;
  }
  CUtensorMap mA, mB;
  {
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)nrhs};   // k beyond n: TMA zero fill
    cuuint64_t strides[1] = {(cuuint64_t)ldg};
    cuuint32_t box[2] = {TK, TM};
    int rc = encode(&mA, 2, G, dims, strides, box);
    if (rc != GG_OK) return rc;
  }
  CUtensorMap mB1;
  {   // tile-packed slices [tile][slice][row][k]: boxes of 3 slices x 32 rows and 1 slice x 16
    cuuint64_t dims[4] = {(cuuint64_t)ST, (cuuint64_t)ST, (cuuint64_t)S,
                          (cuuint64_t)slice_tiles(np)};
    cuuint64_t strides[3] = {(cuuint64_t)ST, (cuuint64_t)ST * ST, (cuuint64_t)ST_BYTES};
    cuuint32_t box3[4] = {TK, TR, 3, 1};
    int rc = encode(&mB, 4, Sl, dims, strides, box3);
    if (rc != GG_OK) return rc;
    cuuint32_t box1[4] = {TK, TR / 2, 1, 1};
    rc = encode(&mB1, 4, Sl, dims, strides, box1);
    if (rc != GG_OK) return rc;
  }
  I8Args a;
  a.N = nrhs;
  a.num_rb = np / TR;
  a.num_nt = (nrhs + TM - 1) / TM;
  a.X = X;
  a.ldx = ldx;
  a.expo = expo;
  a.G = G;
  a.ldg = ldg;
  a.n = n;
  a.q = q;
  a.XL = XL;
  a.ldxl = ldxl;
  a.y = y;
  a.P = P;
  a.gate = gate;
  a.gate_value = gate_value;
  // the dynamic tile scheduler's counter lives in the caller's workspace, cleared on the
  // launch stream (stream-ordered with the kernel that uses it)
  GG_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), s));
  a.tile_counter = counter;
  {
    const int pairs = (a.num_rb / 2) * ((a.num_nt + 1) / 2);   // tiles
    int clusters = sms() / 2;
    if (const char* cap = std::getenv("GG_I8_MAX_PAIRS")) {   // tuning / what-if knob
      const int c = std::atoi(cap);
      if (c > 0 && c < clusters) clusters = c;
    }
    if (clusters > pairs) clusters = pairs;
    // SNP groups (tile_coords): ~16 pairs (4,096 SNPs) at n = 10^4, scaled by sqrt(10^4 / n) --
    // the genotype group must stay L2-resident while the row blocks re-read it, and every group
    // re-reads the slices.  Measured DRAM bytes per 8,192-SNP launch (ncu): n = 10^4 2.5 GB
    // (one group) -> 0.83 GB (16 pairs), n = 4*10^4 150 GB -> 43 GB (8 pairs).
    // QUAD tiles (one row block x two SNP pairs) with GG_I8_QUAD=1 (measured r02: config 3
    // +0.6%, within noise; config 1 -1.6% -- the slice bytes are not where the power goes, the
    // multipliers' B-operand bit activity is: profiles/r02_peak_swap.log)
    bool quad = false;
    if (const char* qd = std::getenv("GG_I8_QUAD")) quad = std::atoi(qd) != 0;
    // column units: 256-SNP pairs (dual) or 512-SNP quads (QUAD); the group size is set in pairs
    const int num_cu = quad ? (a.num_nt + 3) / 4 : (a.num_nt + 1) / 2;
    int grp = (int)(16.0 * std::sqrt(1e4 / (double)n) + 0.5);
    if (const char* g = std::getenv("GG_I8_SNP_GROUP")) {   // tuning knob: pairs per group
      const int v = std::atoi(g);
      if (v > 0) grp = v;
    }
    if (quad) grp = (grp + 1) / 2;
    grp = grp < 1 ? 1 : (grp > num_cu ? num_cu : grp);
    const int ngroups = (num_cu + grp - 1) / grp;
    a.grp_pp = (num_cu + ngroups - 1) / ngroups;                // equal-width groups
    a.whatif = 0;
    if (const char* w = std::getenv("GG_I8_WHATIF")) a.whatif = std::atoi(w);
    // A/B knob (bitwise-equal results): GG_I8_EPI=2 forms the dots one chain at a time
    if (const char* e = std::getenv("GG_I8_EPI"))
      if (std::atoi(e) & 2) a.whatif |= 32;
    a.order = 0;
    if (const char* o = std::getenv("GG_I8_ORDER")) a.order = std::atoi(o);   // tuning knob
    a.quad_interleave = 1;
    if (const char* qi = std::getenv("GG_I8_QUAD_ILV")) a.quad_interleave = std::atoi(qi);
    a.rd_bytes = rd_bytes(q, P != nullptr);
    // dual: 5 stages of 44 KB when the row data is small (q <= 3), else 4; QUAD: 4 of 46 KB
    const bool five = !quad && d_smem_bytes(5, a.rd_bytes) <= (size_t)smem_optin();
    auto kern = quad ? trsm_i8_dual_kernel<4, true>
                     : (five ? trsm_i8_dual_kernel<5, false> : trsm_i8_dual_kernel<4, false>);
    const size_t smem = d_smem_bytes(five ? 5 : 4, a.rd_bytes, quad);
    if (smem > (size_t)smem_optin()) {
      set_error("trsm_i8: shared memory for the pipeline exceeds the device limit");
      return GG_ECUDA;
    }
    GG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GG_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mA, mB, mB1, a));
    return GG_OK;
  }
}

}  // namespace gg
