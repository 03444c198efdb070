/*
 * bse200 — C ABI of the B200-native pseudo-hermitian ChASE hot path.
 *
 * Every entry point replaces one operator of the reference Python package
 * `bsesolve` (paths relative to /root/reference/pkg/src/bsesolve/); the
 * Python host layer `paper_2601_10557_b200` binds them with ctypes exactly
 * as a maintainer of the reference would.
 *
 * Conventions
 *   - All matrices are complex128, column-major, interleaved (re, im) —
 *     numpy's `complex128` / F-order, torch's `complex128` column-major.
 *   - Pointers named `d_*` are DEVICE pointers (cudaMalloc / torch CUDA
 *     storage); `h_*` are HOST pointers.  Sizes are int64_t element counts.
 *   - The Hamiltonian operand `d_ab` is the m x 2m device matrix [A | B]
 *     (leading dimension `lda` >= m): A hermitian, B symmetric, exactly the
 *     two blocks `BseHamiltonian` stores (hamiltonian.py:63-96).
 *   - Work is enqueued on the context's stream (bse_set_stream); functions
 *     that return host scalars synchronise that stream.
 *   - Return value: BSE_OK or one of the BSE_E* status codes, which the
 *     Python layer maps onto the reference exception classes
 *     (errors.py:8-38).  bse_last_error() returns the message.
 *   - Deterministic: no atomics in any reduction; reruns are bitwise equal.
 */
#ifndef BSE200_H
#define BSE200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BSE_OK = 0,
  BSE_EVALIDATION = 1,   /* ValidationError            errors.py:12 */
  BSE_ENUMERICAL = 2,    /* NumericalError             errors.py:16 */
  BSE_EINDEFINITE = 3,   /* IndefiniteError            errors.py:20 */
  BSE_ERANK = 4,         /* RankDeficiencyError        errors.py:24 */
  BSE_ELANCZOS = 5,      /* LanczosBreakdownError      errors.py:28 */
  BSE_EHERMITIAN_RQ = 6, /* HermitianRqError           errors.py:32 */
  BSE_ECUDA = 7          /* CUDA / cuSOLVER failure (NumericalError on the Python side) */
};

typedef struct bse_ctx bse_ctx;

/* Hamiltonian flags (bse_set_hamiltonian_flags) */
#define BSE_HAM_B_ZERO 1u /* B == 0 (TDA / hermitian limit): the operator skips the B half (4 n^2 k flops) */

/* ---- context ------------------------------------------------------------ */
int bse_ctx_create(int device, bse_ctx** out);
void bse_ctx_destroy(bse_ctx* ctx);
int bse_set_stream(bse_ctx* ctx, void* cuda_stream);
const char* bse_last_error(const bse_ctx* ctx);
/* number of bse200 kernels launched through this context (evidence counter) */
int64_t bse_launch_count(const bse_ctx* ctx);
const char* bse_version(void);
/* Kernel of the Chebyshev-filter products (and of H products given sum planes): 4 = 4M split
 * (8 real DMMA per complex block pair; the context default); 3M / Gauss (6 DMMA, 25% fewer FP64
 * tensor ops, error bound ~eps (|Re|+|Im|)^2): 88 = TMA-fed producer-warp kernel
 * (the 3M default), 82 / 86 its narrow / wide tiles; without the sum planes the same kernel forms
 * the operand sums in registers (same bits).  90 / 92 / 94 / 96 / 97 / 98: the real-split kernel
 * (csrc/hop_rs.cuh, 4 n^2 k flops per step) for bse_chebyshev_filter_rs, bse_hop_tile_rs(_t) and
 * registered RR planes, 90 = tile and split-K factor by block shape (the Python default),
 * 92 / 94 / 96 / 97 fixed unsplit tiles (bitwise identical), 98 = tile 97 with its K range split
 * over 2 CTAs (env BSE200_RS_KSPLIT overrides the factor; partial sums reduced in a fixed order);
 * complex-operand products run code 88 under them.  BSE_EVALIDATION for other codes.          */
int bse_set_filter_algorithm(bse_ctx* ctx, int complex_mults);
/* Properties of the Hamiltonian the following operator calls on this context act on
 * (BSE_HAM_* flags); the Python layer sets them before every operator call.                     */
int bse_set_hamiltonian_flags(bse_ctx* ctx, unsigned flags);
/* (code 6 = 3M using the precomputed sum planes when the caller passes them)                   */

/* ---- Hamiltonian operator ------------------------------------------------ */
/* y = H x  (low_sign = +1)  or  y = S H x  (low_sign = -1)
 * replaces apply_h hamiltonian.py:132-151 (and apply_s(apply_h(.)) at
 * rayleigh_ritz.py:112).  x, y: n x k (n = 2m), must not alias.
 * d_sd (nullable): the (Pr + Pi, Pr - Pi) planes of d_ab (bse_make_sum_planes); when given, the
 * product runs on the kernel selected by bse_set_filter_algorithm (3M), else on the 4M kernel. */
int bse_apply_h(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_x, int64_t ldx,
                void* d_y, int64_t ldy, int64_t k, double low_sign);

/* One Chebyshev step y_next = alpha (H y - c y) - beta y_prev, fused in the
 * GEMM epilogue (chebyshev.py:68-74).  y_next may alias y_prev, not y.    */
int bse_filter_step(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_y,
                    const void* d_yprev, void* d_ynext, int64_t ld, int64_t k, double c, double alpha, double beta);

/* Whole filter p(H) V (chebyshev.py:51-75): degree `deg` (even) products,
 * sigma-scaled recurrence with c = center, e = half_width, s = scale_ref.
 * d_v (n x k, ld) is overwritten with the result; d_work must hold 2 n x k
 * blocks with the same ld (rotating recurrence buffers).                   */
int bse_chebyshev_filter(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, void* d_v,
                         int64_t ld, int64_t k, int deg, double c, double e, double s, void* d_work);
/* 3M operand sums: d_sd (same shape / lda as d_ab, m x cols) <- (re + im, re - im) of d_ab.
 * Passed as d_sd to the filter entry points, it removes the P-side adds from the 3M kernel's
 * critical path (+32 m^2 bytes).  d_sd may be NULL everywhere (sums formed on the fly).      */
int bse_make_sum_planes(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, int64_t cols, void* d_sd);

/* Real-split filter planes (csrc/hop_rs.cuh): d_g (mr x 4kc doubles, leading dim ldg, even, >= mr)
 * <- [Ai + Bi | Ar - Br | Ar + Br | Ai - Bi] of a tile d_ab = [A_t | B_t] (mr x 2kc complex;
 * mr = kc = m for the whole operator: 32 m^2 bytes, built once).                              */
int bse_make_rs_planes(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t mr, int64_t kc, void* d_g, int64_t ldg);
/* Register real-split planes d_g (bse_make_rs_planes, mr = kc = m) of the operator d_ab on the
 * context: while registered, the T = (S) H Q products of bse_rr_hermitian / bse_rr_backup with
 * this d_ab run on the real-split kernel (fold Q, product, unfold with the S-flip).  d_g = NULL
 * clears the registration (the Python layer scopes it to one RR call).  d_ab may be NULL for an
 * operator held as planes only (one GPU at n = 100k: the planes replace [A|B]); the RR calls
 * then take d_ab = NULL too and every product, k = 1 included, runs on the planes.             */
int bse_set_rs_planes(bse_ctx* ctx, const void* d_ab, int64_t m, const void* d_g, int64_t ldg);
/* Register a device buffer of 4 k^2 complex128 + k doubles that the next bse_rr_hermitian /
 * bse_rr_backup calls fill with their reduced problem (rayleigh_ritz.py:41-51, 140-143, 176-179):
 * [W | L (lower triangle; upper = W's) | M | G] column-major k x k each, then d (backup only).
 * NULL clears it; the solver loop never registers one (no copies on the hot path).             */
int bse_set_rr_capture(bse_ctx* ctx, void* d_buf);
/* bse_chebyshev_filter (chebyshev.py:51-75) on the real-split planes: the block is folded to
 * (X1 + X2, X1 - X2), where H acts through four real m x m planes (4 n^2 k executed flops per
 * step instead of 6 n^2 k for 3M), filtered, and unfolded.  Same arguments and results as
 * bse_chebyshev_filter up to rounding; requires B != 0 (BSE_HAM_B_ZERO unset).              */
int bse_chebyshev_filter_rs(bse_ctx* ctx, const void* d_g, int64_t ldg, int64_t m, void* d_v, int64_t ld, int64_t k,
                            int deg, double c, double e, double s, void* d_work);

/* Residual norms r_j = ||H v_j - lam_j v_j||_2 (rayleigh_ritz.py:182-190),
 * fused residual-norm epilogue; h_lam (k) in, h_res (k) out on host.      */
int bse_residuals(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const void* d_v, int64_t ldv, int64_t k,
                  const double* h_lam, double* h_res);

/* ---- orthonormalisation (ortho.py:96-158) --------------------------------- */
/* In place: project out span(S Y_locked) (Y: n x l, may be l = 0), then
 * CholQR2; on failure shifted CholQR3 (replacing the Householder fallback);
 * then the column phase convention of ortho.py:70-82.
 * *h_method = 0 cholqr2, 1 shifted fallback.  BSE_ERANK on rank deficiency. */
int bse_s_orthonormalize(bse_ctx* ctx, void* d_v, int64_t n, int64_t k, int64_t ldv, const void* d_ylocked,
                         int64_t l, int64_t ldy, int* h_method);
/* Incremental basis of span(S Y_locked): S-flip the c newly locked columns d_ynew into
 * basis[:, l_old:l_old+c], project them twice against basis[:, :l_old] and CholQR them (the
 * reference re-QRs the whole flipped locked block every iteration, ortho.py:149-150; same span). */
int bse_extend_sbasis(bse_ctx* ctx, void* d_basis, int64_t n, int64_t ldb, int64_t l_old, const void* d_ynew,
                      int64_t ldy, int64_t c);
/* ortho.py:132-158 with the locked space given by that orthonormal basis (n x l, leading dim
 * ldb): projection, CholQR2 with the shifted fallback, phase convention; h_method as
 * bse_s_orthonormalize.                                                                       */
int bse_s_orthonormalize_basis(bse_ctx* ctx, void* d_v, int64_t n, int64_t k, int64_t ldv, const void* d_basis,
                               int64_t l, int64_t ldb, int* h_method);
int bse_cholqr(bse_ctx* ctx, void* d_q, int64_t n, int64_t k, int64_t ldq, int* h_method);
/* column phase convention alone (fix_column_phases, ortho.py:70-82) */
int bse_fix_phases(bse_ctx* ctx, void* d_q, int64_t n, int64_t k, int64_t ldq);

/* ---- Rayleigh-Ritz (rayleigh_ritz.py:98-179) ------------------------------ */
/* Hermitian-equivalent oblique RR on the active basis Q (n x k):
 * h_lam (k) ascending Ritz values, d_vout (n x k) unit Ritz vectors,
 * *h_lam_min_m = |lambda|_min(Q*SQ).  BSE_EHERMITIAN_RQ when Q*SQ is
 * singular (< 1e-8), Q*SHQ is not positive definite, or theta ~ 0.
 * h_res (nullable): residual norms ||H v - lam v|| from the RR intermediate,
 * H V = S (S H Q) w / |Q w| (rayleigh_ritz.py:182-190 without a second H product).
 * d_sd (nullable): sum planes of d_ab, as for bse_apply_h (the T = S H Q product). */
int bse_rr_hermitian(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_q,
                     int64_t ldq, int64_t k, double* h_lam, void* d_vout, int64_t ldvout, double* h_lam_min_m,
                     double* h_res);
/* Non-hermitian backup projection (Alg. 3, rayleigh_ritz.py:146-179); d_sd as above. */
int bse_rr_backup(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_q,
                  int64_t ldq, int64_t k, double* h_lam, void* d_vout, int64_t ldvout, double* h_lam_min_m);

/* ---- Lanczos bounds (lanczos.py:53-88) ------------------------------------ */
/* One S-inner-product Lanczos sweep from host start vector h_start (n):
 * h_alpha (steps), h_beta (steps-1); *h_count = number of alphas produced.
 * BSE_EINDEFINITE if the start has non-positive S*H norm.                  */
int bse_lanczos_sweep(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const void* h_start, int steps,
                      double* h_alpha, double* h_beta, int* h_count);

/* ---- input checks --------------------------------------------------------- */
/* Cholesky of the materialised S H (hamiltonian.py:208-218); *h_definite = 1/0. */
int bse_is_definite(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, int* h_definite);

/* ---- building blocks of the 2D-distributed solve (paper_2601_10557_b200/dist.py) ---- */
/* One tile product of the fused H operator with an axpby epilogue:
 *   y_half = low_sign^[half==low] * ( alpha * (P-product_half - shift_r * s_half) - beta * p_half )
 * with U = pa x1 + pb x2 and L' = conj(pa) x2 + conj(pb) x1 (H x = [U; -L']), pa/pb mr x kc tiles.
 * shift_r = d_shift_col[col] (per column, if non-null) or `shift`, applied on output rows
 * [shift_lo, shift_hi) only: the rows a 2D tile's input block shares with its output block
 * (PAPER.md:723-740 communication-avoiding filter).                                            */
typedef struct {
  const void* pa;
  const void* pb;
  const void* sa; /* optional 3M sum planes of pa / pb (bse_make_sum_planes), may be NULL */
  const void* sb;
  int64_t lda, mr, kc;
  const void* x1;
  const void* x2;
  int64_t ldx, k;
  void* y1;
  void* y2;
  int64_t ldy;
  const void* s1;
  const void* s2;
  int64_t lds, shift_lo, shift_hi;
  double shift;
  const double* d_shift_col;
  const void* p1;
  const void* p2;
  int64_t ldp;
  double alpha, beta, low_sign;
  int filter; /* 1: a Chebyshev-filter product (uses the algorithm set by bse_set_filter_algorithm) */
} bse_hop_tile_args;
int bse_hop_tile(bse_ctx* ctx, const bse_hop_tile_args* args);
/* The tile product of a filter step on the tile's real-split planes d_g (bse_make_rs_planes of
 * [pa | pb]): x1 / x2 are the folded parts (X1 + X2, X1 - X2) of the input rows, y1 / y2 receive
 * the folded halves of the output; low_sign must be 1 (no S-flip); B != 0.  pa / pb / sa / sb are
 * not read.  The 2D-grid filter folds its block once (bse_rs_fold), runs deg such products with
 * the same reductions as bse_hop_tile, and unfolds.                                            */
int bse_hop_tile_rs(bse_ctx* ctx, const bse_hop_tile_args* args, const void* d_g, int64_t ldg);
/* The TRANSPOSED tile product on the same planes d_g: d_g holds the planes of a tile T (kc x mr
 * real, leading dim ldg >= kc, even) and the product is that of the block transpose
 * [A_T^H | B_T^T] (mr output rows = T's columns, contraction kc = T's rows), the row -> col step
 * of the 2D grid (the same local block, conjugate-transposed), so a grid GPU
 * stores one tile's planes.  Arguments and epilogue as bse_hop_tile_rs.                        */
int bse_hop_tile_rs_t(bse_ctx* ctx, const bse_hop_tile_args* args, const void* d_g, int64_t ldg);
/* Fused group reduction of the 2D grid's tile products (dist.py, BSE200_FUSED_REDUCE=1): the next
 * real-split tile products (bse_hop_tile_rs / _rs_t) store their output tile not to y1 / y2 but to
 * each of the n (<= 4) base pointers -- this rank's slot in every group member's symmetric
 * (NVLink peer-mapped) inbox, same layout as y -- from the kernel epilogue, so the transfer
 * overlaps the product tile by tile; n = 0 restores local output.  Replaces the NCCL allreduce
 * after the tile product (dist.py sum_row / sum_col; the paper's row / column allreduce,
 * PAPER.md:723-740).                                                                           */
int bse_set_push_targets(bse_ctx* ctx, void* const* y_bases, int n);
/* y[i] = sum_{j < nslot} inbox[j * slot_stride + i], i < count (complex elements), slots added in
 * order: the second half of the fused group reduction, after a barrier among the group.        */
int bse_group_sum(bse_ctx* ctx, const void* d_inbox, int64_t slot_stride, int nslot, void* d_y, int64_t count);
/* (X1, X2) -> (scale (X1 + X2), scale2 (X1 - X2)) for a block of 2 rows x k (ld >= 2 rows; X1 rows
 * [0, rows), X2 rows [rows, 2 rows)); (1, 1) folds, (1/2, 1/2) unfolds, (1/2, -1/2) unfolds with
 * the S-flip; d_dst may equal d_src.                                                           */
int bse_rs_fold(bse_ctx* ctx, const void* d_src, void* d_dst, int64_t ld, int64_t rows, int64_t k, double scale,
                double scale2);
/* CholQR factor step (ortho.py:115-119): hermitise the summed Gram d_g (k x k), add shift I,
 * R = chol upper (in d_g), |diag R| -> d_rdiag (nullable), R^{-1} -> d_rinv; *h_info > 0 on failure. */
int bse_chol_rinv(bse_ctx* ctx, void* d_g, int64_t k, double shift, void* d_rinv, double* d_rdiag, int* h_info);
/* Small pencil of the hermitian RR (rayleigh_ritz.py:113-137) from the summed W = Q^H S H Q
 * and G2 = Q2^H Q2: ascending Ritz values (host) and the sorted back-transform L^{-H} y (device). */
int bse_rr_pencil(bse_ctx* ctx, void* d_w, void* d_g2, int64_t k, double* h_lam, void* d_wvec, double* h_lam_min_m);
/* The two independent halves of bse_rr_pencil, for two GPUs of a grid to solve concurrently:
 * part 1 only writes |lambda|_min(M) to *h_lam_min_m (no check; h_lam / d_wvec unused);
 * part 2 is the pencil without the eigenvalues of M (the caller checks |lambda|_min(M) >= 1e-8
 * first, as rayleigh_ritz.py:116-126 orders the errors).                                        */
int bse_rr_pencil_part(bse_ctx* ctx, int part, void* d_w, void* d_g2, int64_t k, double* h_lam, void* d_wvec,
                       double* h_lam_min_m);
/* Small problem of the backup RR (rayleigh_ritz.py:160-175) from summed partials G0 = Q^H S H Q
 * (overwritten), W = Q^H H Q and G2 = Q2^H Q2 (overwritten), all k x k: ascending real parts of the
 * eigenvalues (host) and the matching eigenvectors y (device, k x k); V = Q y / |Q y| is the caller's. */
int bse_rr_backup_pencil(bse_ctx* ctx, void* d_g0, const void* d_w, void* d_g2, int64_t k, double* h_lam, void* d_y,
                         double* h_lam_min_m);
/* residual partials from the RR intermediate: out[j] = sum_i |sgn_i u_ij uscale_j - lam_j v_ij|^2,
 * sgn_i = -1 for rows >= half (u = (S H Q) w, v = unit Ritz vectors, uscale = 1/|Q w|)            */
int bse_resid_partial(bse_ctx* ctx, const void* d_u, int64_t ldu, const void* d_v, int64_t ldv, int64_t rows,
                      int64_t half, int64_t k, const double* d_uscale, const double* d_lam, double* d_out);
/* squared column norms of a rows x k block (device out); x /= sqrt(norm2) per column           */
int bse_colnorm2(bse_ctx* ctx, const void* d_x, int64_t rows, int64_t k, int64_t ldx, double* d_out);
int bse_colscale_rsqrt(bse_ctx* ctx, void* d_x, int64_t rows, int64_t k, int64_t ldx, const double* d_norm2);
/* max |G - I| of a k x k device matrix (ortho.py:124)                                         */
int bse_defect(bse_ctx* ctx, const void* d_g, int64_t k, double* h_out);
/* y = S x for a block of 2*half rows (rows >= half negated)                                   */
int bse_sflip(bse_ctx* ctx, const void* d_x, int64_t ldx, void* d_y, int64_t ldy, int64_t half, int64_t k);

/* ---- complex64 filter on the tcgen05 tensor cores (configs[4] c64 variant) ---------------
 * d_pplanes: 4 fp32 planes (Re hi, Re lo, Im hi, Im lo) of [A | B] in the K-major layout
 * [m rows][2 mp] (mp = m rounded up to 4), i.e. 32 m mp bytes, built by bse_c64_prepare.
 * bse_chebyshev_filter_c64: p(H) v with FP32-accurate 3xTF32 tcgen05.mma products, the
 * recurrence in FP32 (chebyshev.py:51-75); d_v (complex128 n x k) in/out; d_work: 48 mp k floats. */
int bse_c64_prepare(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, void* d_pplanes);
int bse_chebyshev_filter_c64(bse_ctx* ctx, const void* d_pplanes, int64_t m, void* d_v, int64_t ldv, int64_t k, int deg,
                             double c, double e, double s, void* d_work);

/* complex64 filter on a tile of the 2D grid (dist.py).  A "plane set" of an n = 2 rows x k block
 * is 8 consecutive fp32 planes (Re hi, Re lo, Im hi, Im lo, then their negations) of
 * 2 pad4(rows) k floats each (column-major, lower half at row pad4(rows)).
 * bse_c64_tile_planes: the 4 P planes of a tile with output rows mo and contraction kc per part,
 *   read from the columns of the transposed blocks (src_a = A^H block, src_b = B^T block, kc x mo,
 *   leading dim lds): the fwd tile's planes come from the trn tile and vice versa.
 * bse_c64_tile_step: out = alpha (tile x - shift x[rows + s_off] on rows [shift_lo, shift_hi))
 *   - beta prev; raw != 0 writes the unsplit fp32 Re / Im planes (2 planes) for an allreduce,
 *   bse_c64_split turns them into the next step's plane set.                                   */
typedef struct {
  const void* pplanes; /* bse_c64_tile_planes of this tile */
  int64_t mo, kc, k;   /* output rows per half, contraction per part (input rows per half), columns */
  const void* x;       /* input plane set (kc rows per half) */
  const void* prev;    /* y_prev plane set (mo rows; nullable when beta == 0) */
  void* out;           /* output plane set, or the 2 raw planes when raw != 0 */
  double alpha, beta, shift;
  int64_t shift_lo, shift_hi, s_off;
  int raw;
} bse_c64_tile_args;
int bse_c64_tile_planes(bse_ctx* ctx, const void* d_src_a, const void* d_src_b, int64_t lds, int64_t mo, int64_t kc,
                        void* d_pplanes);
int bse_c64_tile_step(bse_ctx* ctx, const bse_c64_tile_args* args);
int bse_c64_split(bse_ctx* ctx, const void* d_raw, int64_t rows, int64_t k, void* d_planes);
int bse_c64_to_planes(bse_ctx* ctx, const void* d_v, int64_t ldv, int64_t rows, int64_t k, void* d_planes);
int bse_c64_from_planes(bse_ctx* ctx, const void* d_planes, int64_t rows, int64_t k, void* d_v, int64_t ldv);

/* ---- synthetic inputs (generate.py:60-83 on the device) -------------------- */
/* complex normals start_index .. +count of stream `seed` (rng.py:63-81):
 * bit-exact splitmix64 words, device libm Box-Muller (<= ~1 ulp from host). */
int bse_complex_normals(bse_ctx* ctx, void* d_out, uint64_t seed, int64_t start_index, int64_t count);
/* the transpose (cols x rows, column-major) of the rows x cols normal matrix */
int bse_complex_normals_t(bse_ctx* ctx, void* d_out, uint64_t seed, int64_t rows, int64_t cols);
/* a <- (a + a^T)/2 (conj = 0) or (a + a^H)/2 (conj = 1), m x m              */
int bse_symmetrize(bse_ctx* ctx, void* d_a, int64_t m, int64_t lda, int conj);
/* a <- scale * (conj ? conj(a) : a) + shift * I                             */
int bse_scale_shift(bse_ctx* ctx, void* d_a, int64_t m, int64_t lda, double scale, double shift, int conj);
/* eigenvalues (ascending, host) of a hermitian device matrix                */
int bse_eigvalsh(bse_ctx* ctx, const void* d_a, int64_t k, int64_t lda, double* h_w);

/* ---- generic tall-skinny products (also used by tests) -------------------- */
/* C = alpha * A^H B + beta C  (A: K x M, B: K x N)   */
int bse_zgemm_cn(bse_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const void* d_a, int64_t lda,
                 const void* d_b, int64_t ldb, double beta, void* d_c, int64_t ldc);
/* C = alpha * A B + beta C    (A: M x K, B: K x N)   */
int bse_zgemm_nn(bse_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const void* d_a, int64_t lda,
                 const void* d_b, int64_t ldb, double beta, void* d_c, int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif /* BSE200_H */
