/*
 * gwasgls_b200.h — C-ABI of the B200-native GLS hot path (libgwasgls_b200.so).
 *
 * This is the drop-in boundary for the reference package `gwasgls` (pure Python,
 * /root/reference/pkg/src/gwasgls).  The reference has no FFI of its own: its
 * boundary is the module namespace `gwasgls.kernel`.  Each entry
 * point below replaces one function of that namespace (cited per function); the
 * Python host layer `paper_1304_2272_b200.kernel` binds them with ctypes and keeps
 * the reference's names, signatures and exceptions.  INTEGRATION.md shows the
 * reference-side binding.
 *
 * Conventions (all entry points):
 *   - Return an int status: GG_OK, or one of the GG_E* codes; gg_last_error()
 *     returns the message of the calling thread's last failure.
 *   - Pointers are DEVICE pointers on the calling thread's current CUDA device,
 *     unless named *_host.  `stream` is a cudaStream_t (NULL = legacy default).
 *   - All matrices are column-major FP64 ("F-order", like the reference's
 *     buffers, pipeline.py:195).  Every matrix whose rows run over the n
 *     individuals is stored with its rows padded to np = gg_pad(n) (a multiple of
 *     GG_TILE) and leading dimension >= np.  Padding rows of right-hand sides
 *     are zero; L and Linv are extended by the identity on the padding block.
 *     Column counts are never padded.
 *   - No entry point allocates persistent device memory; workspaces (including the int8
 *     TRSM's tile counter) come from the caller (sizes from the *_workspace_bytes queries).
 *     The one handle is gg_dist_comms (created by gg_dist_comms_*, owned by the caller,
 *     released by gg_dist_comms_free: NCCL communicators or transport callbacks).
 *     The only process-wide state is the once-resolved cuTensorMapEncodeTiled pointer.
 *     Entry points are reentrant and keep no unguarded global state (SPEC threading rule,
 *     SURVEY §8b).
 */
#ifndef GWASGLS_B200_H
#define GWASGLS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GG_OK 0
#define GG_ENOTPD 1      /* Cholesky pivot <= 0 / NaN, or non-finite input      */
#define GG_EDIM 2        /* inconsistent sizes / leading dimensions              */
#define GG_ECUDA 3       /* CUDA runtime error                                   */
#define GG_ENCCL 4       /* a failed collective (gg_dist_*: NCCL or a transport callback); the
                            host layer (comm.py) raises TransportFailure with this meaning     */
#define GG_EARG 5        /* invalid argument (NULL pointer, unsupported p, ...)  */

#define GG_TILE 128      /* row padding unit = GEMM tile edge                    */
#define GG_PMAX 20       /* largest p supported by the small-system solver       */
#define GG_STATUS_INVALID (-2) /* per-SNP status: block not computable on the chosen path */
#define GG_DOT_BLOCK 32  /* rows per partial sum of the canonical reduction order */

/* Library identification / errors. */
const char* gg_version(void);
const char* gg_last_error(void);
int gg_pad(int n);                               /* round n up to GG_TILE          */

/* ---- Cholesky + triangular inverse ------------------------------------------------
 * Replaces kernel.cholesky_spd (kernel.py:92-109: LAPACK dpotrf lower, clean=1,
 * input untouched) and produces, in the same pass, Linv = L^-1 (the operand of the
 * streamed TRSM, see gg_trsm_lower_f64).
 *   M      : n x n, leading dimension ldm (>= n); only read.  m_row_major = 1 reads M in
 *            row-major order (a C-contiguous numpy array uploaded as is), 0 column-major.
 *   L      : np x np output, ld = ldp (>= np, multiple of 2); lower factor, upper zero.
 *   Linv   : np x np output, ld = ldp; lower inverse, upper zero.
 *   work   : gg_potrf_workspace_bytes(n) bytes of device scratch (includes the int8
 *            slices of the Ozaki-scheme updates: ~0.6 GB at n = 1e4, ~5.8 GB at 4e4).
 * The large trailing SYRKs and inverse updates run as FP64 GEMMs on the int8 tensor
 * cores (gg_gemm_ozaki_f64, FP64-GEMM accuracy); GG_FACTOR_OZAKI=0 selects DMMA.
 *   info_host[0] : -1 on success, else the 0-based failing pivot (LAPACK info-1, or
 *                  for non-finite input the row of the first non-finite entry in
 *                  row-major order, kernel.py:101-103).
 *   info_host[1] : 1 iff the failure was a non-finite entry.
 * Returns GG_ENOTPD on failure.  Synchronises `stream` (to read the pivot).      */
size_t gg_potrf_workspace_bytes(int n);
int gg_potrf_f64(int n, const double* M, int ldm, int m_row_major, double* L, double* Linv,
                 int ldp, void* work, int* info_host, void* stream);

/* Triangular inverse of an arbitrary lower-triangular L (np x np, padded as above,
 * upper part ignored).  Used by kernel.trsolve_lower (kernel.py:112-121) when the
 * caller hands in an L that did not come from gg_potrf_f64.                      */
size_t gg_trtri_workspace_bytes(int n);
int gg_trtri_lower_f64(int n, const double* L, int ldl, double* Linv, int ldp,
                       void* work, void* stream);

/* Blocked forward substitution X = L^-1 B for an arbitrary lower-triangular L (np x np, padded
 * as above, upper part ignored) -- the drop-in kernel.trsolve_lower (kernel.py:112-121: scipy
 * solve_triangular -> dtrtrs -> dtrsm).  The 128 x 128 diagonal blocks are inverted in one
 * launch, then per block column X_J = L_JJ^-1 B_J and B_{J+1:} -= L_{J+1:,J} X_J on DMMA GEMMs:
 * O(n^2 nrhs), backward-stable like dtrsm's blocked form (no O(n^3) explicit inverse).  X may
 * alias B.  work: gg_trsm_lower_blocked_workspace_bytes(n, nrhs) bytes.                        */
size_t gg_trsm_lower_blocked_workspace_bytes(int n, int nrhs);
int gg_trsm_lower_blocked_f64(int n, int nrhs, const double* L, int ldl, const double* B,
                              int ldb, double* X, int ldx, void* work, void* stream);

/* ---- Streamed TRSM -----------------------------------------------------------------
 * X = L^-1 B for nrhs columns, computed as the lower-triangular product Linv * B
 * on FP64 DMMA tiles (replaces kernel.trsolve_lower, kernel.py:112-121, i.e.
 * scipy solve_triangular -> dtrtrs -> dtrsm).  B (ldb) and X (ldx) have np rows
 * (padding rows of B zero); X must not alias B.  Per-column arithmetic is
 * identical for every column position (column-permutation bitwise invariance,
 * tests/test_kernel.py:228-241).                                                   */
int gg_trsm_lower_f64(int n, int nrhs, const double* Linv, int ldp, const double* B,
                      int ldb, double* X, int ldx, void* stream);

/* The production TRSM: same product with the inverse stored ROW-major (LinvT: element
 * (i, k) of Linv at LinvT[k + i*ldp], upper part zero) so both operands are K-major.
 * Persistent warp-specialised kernel: TMA (cp.async.bulk.tensor, 128B swizzle) into a
 * 6-stage mbarrier ring, DMMA consumers.  Bitwise identical to gg_trsm_lower_f64.
 * Operands 16-byte aligned; padding rows of B zero.                                     */
int gg_trsm_lower_rm_f64(int n, int nrhs, const double* LinvT, int ldp, const double* B,
                         int ldb, double* X, int ldx, void* stream);

/* The packed layout of the inverse used by the streamed sweep: only the 128 x 16 tiles on or
 * below the diagonal, tile-major (tile (mt, kt), kt < 8*(mt+1), at index 4*mt*(mt+1) + kt;
 * each tile 128 rows x 16 k, k contiguous).  Half the memory of the square inverse (the
 * 150,000^2 inverse of BASELINE config 4 fits one GPU: 90 GB), and one 3-D TMA box per tile.
 * gg_pack_lower_f64 converts a column-major (row_major = 0) or row-major (1) square inverse. */
size_t gg_packed_lower_bytes(int n);
int gg_pack_lower_f64(int n, const double* A, int lda, int row_major, double* LinvP,
                      void* stream);
int gg_trsm_lower_packed_f64(int n, int nrhs, const double* LinvP, const double* B, int ldb,
                             double* X, int ldx, void* stream);

/* Distributed (BASELINE config 4) assembly: write this rank's share of a 2D block-cyclic
 * lower inverse (block nb, a multiple of 128; grid gr x gc; rank at (prow, pcol); local
 * column-major, leading dimension ldloc) into a full packed buffer, zeros elsewhere.  The
 * all-reduce sum of every rank's buffer is the packed inverse (disjoint supports: exact).
 * Replaces the replicated-panel gathers of distgrid.py:215-233 / 317-320.                  */
int gg_pack_lower_blockcyclic_f64(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                                  const double* Bloc, int ldloc, double* LinvP, void* stream);

/* ---- The int8 tensor-core TRSM for dosage blocks ------------------------------------------
 * Dosages are exact int8, so X = L^-1 G runs on tcgen05.mma.kind::i8 with the inverse split
 * error-free into gg_i8_slices() (= 7) int8 slices per row plus an integer diagonal head:
 *     Linv[i,k] = 2^e_i ( [k == i] h_i + sum_{s=0..6} a_s[i,k] 2^(-7 (s+1)) ),  a_s in [-128, 127]
 * with e_i = max(e_off_i, e_diag_i - 20) (|Linv[i,k]| < 2^e_off_i over k < i, |Linv_ii| <
 * 2^e_diag_i), |h_i| < 2^20; slices 0-5 floor (exact remainders: only slice 0 carries the sign,
 * the others are non-negative), the last rounds to nearest (clipped to 127): the residual is zero-mean and <= 2^(e_i - 50), i.e. 50 bits below the row's largest
 * off-diagonal entry and >= 54 bits below its largest entry whenever the diagonal is >= 16x the
 * off-diagonal maximum (kinship-type covariances).  Each slice product is an exact
 * int32 integer; the head term h_i g_i and the seven products are combined exactly into two
 * int64 halves and rounded once to double (correctly rounded; per-column results independent of
 * the column's position).
 * Slice metadata ("expo" below): gg_slice_meta_ints(n) = 2 np ints, e_i (np) then h_i (np).
 *   gg_slice_inverse_i8 : row-major inverse LinvT (see gg_trsm_lower_rm_f64) -> slices
 *                         (gg_inverse_slices_bytes(n) bytes) + metadata.  Slices are tile-packed:
 *                         the lower triangle of 128 x 128 tiles (row tile mt, k tile kt <= mt)
 *                         at tile index mt (mt+1)/2 + kt, each [slice][row][k] int8 (112 KB):
 *                         3.5 np^2 + O(np) bytes.
 *   gg_slice_packed_inverse_i8 : the same from the packed FP64 inverse of gg_pack_lower_f64.
 *   gg_row_exponents_blockcyclic / gg_slice_meta_i8 / gg_slice_blockcyclic_i8 : the distributed
 *                         form -- each rank computes [e_off | e_diag] (2 np ints) over the blocks
 *                         it owns (INT_MIN where it owns nothing); after a MAX all-reduce
 *                         gg_slice_meta_i8 turns them into the metadata (heads zeroed); each rank
 *                         then writes the slices of the elements it owns (zeros elsewhere) and
 *                         the heads of the diagonals it owns.  SUM all-reduces of the int8 slices
 *                         and of the heads (metadata ints np .. 2np) over disjoint supports are
 *                         exact and give the single-GPU result.
 *   gg_narrow_f64_i8    : FP64 dosages (n x cnt, ldx) -> int8 (n x cnt, ldg; with ldg a multiple
 *                         of 16 the rows up to the next multiple of 16 are zeroed); *bad_dev |= 1
 *                         if any value is not an integer with |v| <= gg_i8_value_bound(n).
 *   gg_trsm_lower_i8    : X (np x nrhs FP64, ldx) = L^-1 G for int8 G (n x nrhs, ldg a multiple
 *                         of 16, 16-byte aligned).                                            */
int gg_i8_slices(void);
/* Largest |value| of an int8 operand for which the int32 slice products stay exact at this n:
 * min(127, floor((2^31 - 1) / (128 n))) -- 127 up to n = 132,104; genotype dosages (<= 2) are
 * exact for n < 8.4e6.  gg_narrow_f64_i8 and gg_gls_block_f64 enforce it (larger values take the
 * FP64 path); callers of gg_trsm_lower_i8* must respect it.                                  */
int gg_i8_value_bound(int n);
size_t gg_inverse_slices_bytes(int n);
int gg_slice_inverse_i8(int n, const double* LinvT, int ldp, int8_t* slices, int* expo,
                        void* stream);
int gg_slice_packed_inverse_i8(int n, const double* LinvP, int8_t* slices, int* expo,
                               void* stream);
size_t gg_slice_meta_ints(int n);
int gg_row_exponents_blockcyclic(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                                 const double* Bloc, int ldloc, int* ex2, void* stream);
int gg_slice_meta_i8(int n, const int* ex2, int* expo, void* stream);
int gg_slice_blockcyclic_i8(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                            const double* Bloc, int ldloc, int* expo, int8_t* slices,
                            void* stream);
int gg_narrow_f64_i8(int n, int cnt, const double* X, long long ldx, int8_t* G, long long ldg,
                     int* bad_dev, void* stream);
/* work: gg_trsm_i8_workspace_bytes() bytes of device memory (the dynamic tile scheduler's
 * counter, cleared on `stream` before the launch); one workspace per in-flight launch.       */
size_t gg_trsm_i8_workspace_bytes(void);
int gg_trsm_lower_i8(int n, int nrhs, const int8_t* slices, const int* expo, const int8_t* G,
                     long long ldg, double* X, int ldx, void* work, void* stream);

/* The same kernel with the per-SNP reductions fused into its TMEM epilogue: writes the
 * canonical-order partial dots P (gg_partials_bytes(n, cnt, q) bytes; Xbar against XLbar (q
 * columns, ld gg_pad(n)) and ybar) and, if X != NULL, Xbar itself.  gate != NULL: the kernel
 * runs only if *gate == gate_value (device-side path selection).
 * gg_gls_reduce_solve_f64 then sums the partials in order and solves each SNP's p x p system
 * (the second half of gg_gls_epilogue_f64).                                                    */
size_t gg_partials_bytes(int n, int cnt, int q);
int gg_trsm_lower_i8_partials(int n, int cnt, const int8_t* slices, const int* expo,
                              const int8_t* G, long long ldg, int q, const double* XLbar,
                              const double* ybar, double* P, double* X, int ldx, const int* gate,
                              int gate_value, void* work, void* stream);   /* work: as above */
int gg_gls_reduce_solve_f64(int n, int cnt, int q, const double* P, const double* S_TL,
                            const double* b_T, double* beta, int* status, double* sinv,
                            void* stream);

/* Square transpose (np x np, np a multiple of 32): T = A^T (column-major both).
 * Turns the Linv produced by gg_potrf_f64 into the LinvT operand above.              */
int gg_transpose_f64(int np, const double* A, int lda, double* T, int ldt, void* stream);

/* General FP64 DMMA GEMM on padded operands: C = alpha*A*op(B) + beta*C with
 * A: m x k (lda), op(B) = B (k x ncols, ldb) or B^T (B stored ncols x k, ldb).
 * m and k must be multiples of GG_TILE and 16; ncols arbitrary (>= 1; a multiple of
 * GG_TILE when trans_b).  Exposed for tests and the kinship generator.            */
int gg_dgemm_f64(int m, int ncols, int k, double alpha, const double* A, int lda,
                 const double* B, int ldb, int trans_b, double beta, double* C, int ldc,
                 void* stream);

/* FP64 GEMM on the int8 tensor cores (Ozaki scheme, 7 slices of balanced 8-bit digits per
 * operand, 28 exact int32 slice products, one rounding): C = beta*C + alpha * A~ B~^T with
 * A~(i,k) = A[i*a_rs + k*a_cs] (m x k) and B~(j,k) = B[j*b_rs + k*b_cs] (ncols x k;
 * B == NULL: B~ = the first ncols rows of A~, ncols <= m).  flags: 1 = A~ lower triangular (A~(i,k) = 0 for k > i),
 * 2 = B~(j,k) = 0 for k < j, 4 = only the tiles on/below the diagonal of C.
 * Accuracy: ~2^-56 of |A~(i,:)|max |B~(j,:)|max per product term (FP64-GEMM order).
 * The factorisation's large updates use it (gg_potrf_f64, gg_trtri_lower_f64; set
 * GG_FACTOR_OZAKI=0 for the DMMA path).  work: gg_gemm_ozaki_workspace_bytes bytes.  */
size_t gg_gemm_ozaki_workspace_bytes(int m, int ncols, int k, int b_is_a);
int gg_gemm_ozaki_f64(int m, int ncols, int k, const double* A, long long a_rs,
                      long long a_cs, const double* B, long long b_rs, long long b_cs,
                      double* C, long long ldc, double alpha, double beta, int flags,
                      void* work, size_t work_bytes, void* stream);

/* ---- Genotype widening -------------------------------------------------------------
 * int8 dosages {0,1,2} (n x cnt, ldg) -> FP64 (np x cnt, ldx), padding rows zeroed.
 * Replaces the FP64 load of BlockReader._load (fileio.py:218-229) for the int8
 * genotype stream (BASELINE config 2).                                             */
int gg_widen_i8_f64(int n, int cnt, const int8_t* G, long long ldg, double* X, int ldx,
                    void* stream);

/* ---- Per-SNP reductions and small SPD solves ----------------------------------------
 * dots[j*(q+2) + k] = sum_i Xbar[i,j]*XLbar[i,k]  (k < q)      (kernel.py:266-267)
 * dots[j*(q+2) + q] = sum_i Xbar[i,j]^2                          (kernel.py:268)
 * dots[j*(q+2)+q+1] = sum_i Xbar[i,j]*ybar[i]                    (kernel.py:269)
 * One fixed summation order for every column: FMA chains over blocks of GG_DOT_BLOCK rows,
 * block sums strided over 32 lanes then an xor butterfly (replaces _column_sums,
 * kernel.py:260-270, and kernel.gram, kernel.py:124-131).                               */
int gg_gls_dots_f64(int n, int cnt, int q, const double* Xbar, int ldx,
                    const double* XLbar, int ldxl, const double* ybar, double* dots,
                    void* work, void* stream);   /* work: gg_partials_bytes(n, cnt, q) bytes */

/* Batched small SPD solve (replaces kernel.cholesky_solve_batch, kernel.py:138-208):
 * S (batch x p x p, row-major per system), rhs (batch x p) -> x (batch x p; NaN rows
 * for failed systems), status (batch; -1 ok, else first failing pivot j),
 * sinv_packed (batch x p(p+1)/2 in np.tril_indices order, or NULL).  2 <= p <= 20
 * (p = 1 allowed).                                                                  */
int gg_small_spd_solve_f64(int batch, int p, const double* S, const double* rhs,
                           double* x, int* status, double* sinv_packed, void* stream);

/* Fused epilogue (replaces kernel.solve_whitened_block's arithmetic,
 * kernel.py:273-294): reductions above + assembly of S = [[S_TL, S_BL^T],[S_BL, S_BR]],
 * rhs = [b_T, b_B] + the small SPD solve.  S_TL (q x q row-major), b_T (q) device.
 * beta (cnt x p), status (cnt), sinv (cnt x p(p+1)/2 or NULL).                      */
int gg_gls_epilogue_f64(int n, int cnt, int q, const double* Xbar, int ldx,
                        const double* XLbar, int ldxl, const double* ybar,
                        const double* S_TL, const double* b_T, double* beta, int* status,
                        double* sinv, void* work, void* stream);   /* work: as gg_gls_dots_f64 */

/* One streamed block end to end (replaces kernel.gls_solve_block, kernel.py:315-342).
 * Paths (all selected PER COLUMN on the device, without a host synchronisation):
 *   slices given, G8 (int8 dosages) : int8 tensor-core TRSM with the per-SNP reductions fused
 *                                     into its TMEM epilogue (Xbar never written) -> solve;
 *   slices given, X64 (FP64)        : device narrowing; a column of exact integers within
 *                                     gg_i8_value_bound(n) takes the int8 path, any other column
 *                                     the FP64 DMMA TRSM (LinvP) -- decided from that column's
 *                                     values alone, so a column's result never depends on its
 *                                     neighbours, the block size or the shard layout;
 *   no slices                       : [widen int8 ->] FP64 DMMA TRSM (LinvP) -> reductions.
 * Without LinvP (slices only: the config-4 form) a column the int8 path cannot compute exactly
 * gets status GG_STATUS_INVALID and NaN coefficients.
 * Then the batched p x p solve.  XLbar has leading dimension gg_pad(n).  work: at least
 * gg_gls_block_workspace_bytes(n, q, cnt, input_int8, have_slices) bytes of device memory.   */
size_t gg_gls_block_workspace_bytes(int n, int q, int cnt, int input_int8, int have_slices);
int gg_gls_block_f64(int n, int q, int cnt, const double* LinvP, const int8_t* slices,
                     const int* expo, const double* XLbar, const double* ybar,
                     const double* S_TL, const double* b_T, const double* X64, int ldx,
                     const int8_t* G8, long long ldg, void* work, double* beta, int* status,
                     double* sinv, void* stream);

/* ---- Stream plumbing ----------------------------------------------------------------
 * Pitched asynchronous copy (host<->device or device<->device) on `stream`; used by the
 * double-buffered genotype stream (pinned n x cnt host block -> np-padded device block).
 * kind: 1 = host to device, 2 = device to host, 3 = device to device.                */
int gg_memcpy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                      size_t height, int kind, void* stream);

/* ---- Synthetic BASELINE generator (test / bench data, not on the timed path) ------
 * Counter-based splitmix64 streams (the reference's datagen.py:35-52 construction),
 * bit-identical to paper_1304_2272_b200.datagen on the host.
 * maf[j] = maf_lo + (maf_hi - maf_lo) * U(seed, STREAM_MAF, first + j)
 * G[i, j] = [U(seed, s_geno, (first+j)*n + i) < f] + [U(seed, s_geno, (m+first+j)*n + i) < f]
 * Written as int8 (n x cnt, ldg).  When Z != NULL also writes the standardised
 * Z = (G - 2f)/sqrt(2f(1-f)) as FP64 (np x cnt, ldz, padding rows zero).           */
int gg_gen_genotypes_i8(unsigned long long seed, int stream_maf, int stream_geno, int n,
                        long long m, long long first, int cnt, double maf_lo,
                        double maf_hi, int8_t* G, long long ldg, double* Z, int ldz,
                        void* stream);

/* ---- Distributed Cholesky + inverse (configs too large for one GPU) ------------------
 * SURVEY §8b's distributed C-ABI: one rank per GPU, M 2D block-cyclic (nb x nb blocks on an
 * r x c grid, rank = pr * c + pc, the reference's grid_create rule distgrid.py:43-52).
 * Replaces the factorisation of dist_cholesky (distgrid.py:248-288) and yields the inverse
 * too (the distributed prepare's slices come from it).  Collectives run either on NCCL
 * communicators built here (world from one unique id, process row / column split from it;
 * NCCL resolved from the process at run time, no link-time dependency) or on host callbacks
 * (a reference-contract transport: group 0 world, 1 process row, 2 process column; root /
 * member indices within the group; buffers are device pointers, the stream is synchronised
 * before a callback runs).                                                            */
typedef struct gg_dist_comms gg_dist_comms;
typedef int (*gg_dist_bcast_fn)(void* ctx, int group, void* dev, size_t bytes, int root);
typedef int (*gg_dist_allreduce_fn)(void* ctx, int group, double* dev, size_t count);   /* sum */
int gg_dist_nccl_unique_id(unsigned char* id_out /* 128 bytes */);
int gg_dist_comms_nccl(int rank, int nranks, int grid_r, int grid_c, const unsigned char* id,
                       gg_dist_comms** out);
int gg_dist_comms_callbacks(int rank, int nranks, int grid_r, int grid_c, gg_dist_bcast_fn bcast,
                            gg_dist_allreduce_fn allreduce, void* ctx, gg_dist_comms** out);
int gg_dist_comms_free(gg_dist_comms* c);
/* this rank's share: m_loc x n_loc (row blocks pr, pr + r, ...; column blocks pc, pc + c, ...) */
int gg_dist_local_dims(int n, int nb, const gg_dist_comms* c, int* m_loc, int* n_loc);
size_t gg_dist_potrf_workspace_bytes(int n, int nb, const gg_dist_comms* c);
/* Fused distributed Cholesky + inverse.  A: this rank's share of M (column-major, lda >=
 * m_loc; blocks past n hold the identity), overwritten with its share of L (strictly upper
 * blocks zeroed); B: its share of the identity, overwritten with its share of L^-1.  nb a
 * multiple of 128.  Per block column: the diagonal owner factors + inverts (gg_potrf_f64's
 * path) and broadcasts status and inverse over the world; the panel is formed on process
 * column K%c and broadcast along process rows; panel rows for the trailing columns by one SUM
 * all-reduce along process columns; the inverse's block row on process row K%r, broadcast
 * along process columns; local updates on the tensor cores (Ozaki int8 GEMM when every
 * dimension >= 512, DMMA otherwise) with depth-1 look-ahead on a lower-priority side stream.
 * GG_ENOTPD with *info = the global failing column on every rank; GG_ENCCL on a failed
 * collective.  Synchronises `stream` once per block column (the pivot status).            */
int gg_dist_potrf_f64(int n, int nb, double* A, long long lda, double* B, long long ldb,
                      const gg_dist_comms* c, void* work, size_t work_bytes, int* info,
                      void* stream);
/* Distributed TRSM X = L^-1 X (replaces dist_trsolve, distgrid.py:291-314) for L in the
 * block-cyclic share of gg_dist_potrf_f64 and a REPLICATED right-hand side X (padded n x nrhs,
 * ldx >= nblk * nb, rows >= n zero; overwritten with the solution on every rank): blocked
 * forward substitution -- process row K%r forms its partial product of the solved blocks
 * (SUM all-reduce along the process row), the diagonal owner applies its block's inverse
 * (gg_trtri_lower_f64's path) and broadcasts X_K over the world.  Backward-stable.        */
size_t gg_dist_trsm_workspace_bytes(int n, int nb, int nrhs, const gg_dist_comms* c);
int gg_dist_trsm_f64(int n, int nb, int nrhs, const double* L, long long lda, double* X,
                     long long ldx, const gg_dist_comms* c, void* work, size_t work_bytes,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GWASGLS_B200_H */
