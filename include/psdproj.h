/*
 * psdproj.h -- C ABI of the B200-native approximate PSD-cone projection
 * (arXiv:1912.02767, Rontsis, Goulart & Nakatsukasa; PAPER.md in the reference tree).
 *
 * One call projects a symmetric fp64 matrix A onto the PSD cone,
 *     Pi(A) = argmin_{X >= 0} ||A - X||_F = V+ L+ V+^T = A - V- L- V-^T
 * computing only the smaller one-sided eigenspace with warm-started LOBPCG (Alg. 3,
 * PAPER.md:398-412), certifying it with the Theorem-3 residual bound, and
 * choosing the side with the one-third rule. All arithmetic runs in sm_100a
 * kernels on the caller's stream; there is no CPU fallback.
 *
 * Conventions for every entry point:
 *   - Matrices are fp64, column-major, DEVICE pointers unless the name says _host.
 *     A must be exactly symmetric in storage (full storage, both triangles).
 *     Since A is symmetric, row- and column-major are the same.
 *   - lda/ldpi >= n. Pi may alias A (in-place projection) when ldpi == lda.
 *   - The caller owns A, Pi and the workspace (sized by psdproj_workspace_bytes, cuBLAS
 *     style). The context keeps pointers into the workspace; the warm block lives there.
 *     psdproj_destroy frees only the host-side context, never caller memory.
 *   - stream is a cudaStream_t passed as void* (NULL = legacy default stream). Calls are
 *     stream-ordered and return when the info struct is final (host-synchronous).
 *   - A context is used by one host thread and one stream at a time; distinct contexts may
 *     run concurrently.
 *   - Return codes: PSDPROJ_OK (0), PSDPROJ_NOT_CONVERGED (1: Pi and its bound are valid, the
 *     per-pair residual test did not pass within max_iter), negative values are errors;
 *     psdproj_last_error() gives a thread-local message. After E_CUDA the context is
 *     poisoned and must be destroyed.
 */
#ifndef PSDPROJ_H
#define PSDPROJ_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PSDPROJ_OK = 0,
  PSDPROJ_NOT_CONVERGED = 1,
  PSDPROJ_E_INVALID = -1,    /* bad argument; state untouched                               */
  PSDPROJ_E_NONFINITE = -2,  /* A holds inf/nan (detected in the first pass)                */
  PSDPROJ_E_CUDA = -3,       /* CUDA runtime error; context poisoned                         */
  PSDPROJ_E_DEGENERATE = -4, /* pencil not positive definite after dropping P (R20)          */
  PSDPROJ_E_NCCL = -5,       /* reserved for the row-sharded mode                            */
  PSDPROJ_E_WORKSPACE = -6,  /* workspace too small / misaligned (needs 256-byte alignment)  */
  PSDPROJ_E_CAPACITY = -7    /* block width would exceed m_max (no silent fallback)          */
};

enum { PSDPROJ_SIDE_AUTO = 0, PSDPROJ_SIDE_POS = 1, PSDPROJ_SIDE_NEG = -1, PSDPROJ_SIDE_DIRECT = 2 };
enum { PSDPROJ_LOCK_SOFT = 1, PSDPROJ_LOCK_HARD = 2 };

typedef struct psdproj_ctx_s* psdproj_ctx;

typedef struct {
  int max_iter;   /* LOBPCG iteration cap (paper silent, R22); default 500                      */
  int m0;         /* cold block width; 0 => max(ceil(0.1 n), 1) (R28)                          */
  int expand_q;   /* expansion quantum; 0 => max(ceil(0.05 n), 1) (R9)                         */
  int guard;      /* minimum non-positive guard columns (R8, R12); default 1                    */
  int side;       /* PSDPROJ_SIDE_*: 0 = one-third rule                          */
  int locking;    /* PSDPROJ_LOCK_SOFT (BLOPEX active mask) or _HARD (default, R35)             */
  int keep_extra; /* non-positive columns kept in the warm block; <0 => max(guard, ceil(p/10), 16) */
  int m_max;      /* block-width capacity; 0 => ceil(n/3)+1 (wider => DIRECT, R18)              */
  uint64_t seed;  /* Philox4x32-10 key (R11)                                                    */
  uint32_t ctx_id;/* Philox counter word c2 (distinct per cone block)                           */
  int profile;    /* bit 0: time every block-multiply (a3) launch; bit 1: per-phase timing;      */
                  /* bit 2: time every Rayleigh-Ritz tridiagonalisation launch                     */
  int host_io;    /* 1: workspace also holds an n x n staging buffer for psdproj_project_host   */
  int perp_steps; /* f2 (R48): 0 = the paper's bound (perp term ignored); k > 0 =  */
                  /* k-step projected Lanczos upper bound of the perp term added to err_bound     */
  double perp_delta; /* f2: failure probability of that randomized bound (over the Philox start,   */
                     /* Kuczynski-Wozniakowski 1992); 0 => 1e-6                                     */
  double lock_factor; /* hard locking of a positive pair at r <= lock_factor * tol (R55); 0 => 1     */
  int krylov_depth; /* R57 (an extension, NOT the paper's Alg. 3): trial subspace span(X, R, B R, ...,  */
                    /* B^(d-1) R, dX) instead of span(X, R, dX); 0 or 1 => Alg. 3      */
  int guard_active; /* R62: on WARM calls only the guard_active largest non-positive Ritz pairs keep   */
                    /* their residual / dX directions in span(X, R, dX) (the stopping   */
                    /* rule tests the top guard only, R12); 0 => 2; < 0 => every unconverged column   */
                    /* (the BLOPEX active mask of Alg. 3 as printed). Cold calls always use all.      */
  int krylov_max_active; /* R63 (with krylov_depth > 1): the block-Krylov directions of R57 join the   */
                    /* trial subspace only on iterations whose active set J has at most this many     */
                    /* columns (the Rayleigh-Ritz cost grows with the basis width, the fixed launch   */
                    /* latency of an iteration does not); wider active sets use Alg. 3's span(X, R,   */
                    /* dX). 0 => no limit (R57 on every iteration)                     */
} psdproj_params;

typedef struct {
  int status;       /* return code of the call                                                */
  int side;         /* side used: +1, -1, or 2 (DIRECT)                                        */
  int iters;        /* LOBPCG iterations                                                       */
  int m;            /* final block width                                                       */
  int npos;         /* kept pairs (positive Ritz values on the computed side)                  */
  int expansions;   /* random expansions (Alg. 3 line 8)                                       */
  int a_passes;     /* block multiplies B.Z issued                                             */
  int cold;         /* 1 if the call started cold                                              */
  int rr_max;       /* largest Rayleigh-Ritz basis width s                                     */
  int locked;       /* hard-locked columns at exit                                             */
  long long a_cols; /* total columns multiplied by A                                           */
  double err_bound; /* Theorem-3 bound on ||Pi~ - Pi(A)||_F (R14-R16, R36, R53):
                       (1 + e) sqrt(2 ||R+||_F^2 + p^2) + (1 + sqrt 2) d + 7 e theta_max + 4 n u ||A||_F
                       with R+ = B V+ - V+ Theta+ from an explicit B V+ at exit (R16), d =
                       lock_defect, e = orth_defect, p^ = perp_est                           */
  double resid_fro; /* ||R+||_F over the kept pairs (explicit B V+)                           */
  double resid_max; /* max_i r_i over the kept pairs (explicit B V+)                          */
  double lock_defect; /* d = ||V+^T B V+ - diag(theta+)||_F (explicit; hard locking, R36)      */
  double anorm_f;   /* ||A||_F                                                                 */
  double flops;     /* algorithmic flops of the call                           */
  double bytes;     /* algorithmic HBM bytes of the call                                       */
  double amul_flops;/* flops of the block multiplies (2 n^2 sum of columns)                    */
  double amul_bytes;/* bytes of the block multiplies (8 n^2 per pass)                          */
  double amul_ms;   /* summed device time of the block multiplies (profile = 1)                */
  int amul_launches;/* number of timed block-multiply launches                                 */
  int last_pos, last_neg; /* sign counts fed to the next call's side rule                      */
  int launches;     /* kernels this call launched (all of them libpsdproj's own)               */
  int dropped;      /* basis directions dropped at a failing Cholesky pivot (R41)              */
  double phase_ms[12]; /* profile & 2: device time per phase: 0 block multiply, 1 W/P projection,
                         2 Gram/pencil, 3 Cholesky + L^-1 H L^-T, 4 RR tridiagonalisation,
                         5 rotation, 6 residual norms, 7 host round trips / locking / assembly,
                         8 RR bisection, 9 RR inverse iteration, 10 RR back-transformation,
                         11 RR re-orthonormalisation + C' = L^-T Y                          */
  double perp_est;  /* perp term p^ in err_bound: f2 randomized Lanczos bound (R48; 0 if off) or, on
                       the DIRECT path, (1 + e) ||A V- - V- Theta-||_F (R53)                   */
  double orth_defect; /* e = ||V+^T V+ - I||_F of the returned vectors (R53)                   */
  double perp_mu;   /* f2: largest Ritz value of the deflated Lanczos matrix T_k (0 if off)      */
  double tri_ms;    /* profile & 4: summed device time of the RR tridiagonalisation launches      */
  int tri_launches; /* profile & 4: number of timed tridiagonalisation launches                  */
  double tri_flops; /* profile & 4: 4/3 s^3 summed over those launches (algorithmic)              */
  double pi_fro;    /* sqrt(sum of theta+^2): ||Pi(A)||_F on the + side and DIRECT, ||Pi(-A)||_F on
                       the - side (the f3 certificates' PSD-part distances)                      */
} psdproj_info;

/* Fill *p with the defaults documented above. */
void psdproj_default_params(psdproj_params* p);

/* Device workspace needed by a context of order n with these params (NULL = defaults). */
size_t psdproj_workspace_bytes(int n, const psdproj_params* p);

/* Create a context over caller-owned device workspace ws (>= workspace_bytes, 256-B aligned): the
 * state that persists between the projections of one cone block across ADMM iterations -- the warm
 * LOBPCG block (warm starting of multiple Ritz pairs) and the previous sign
 * counts for the one-third rule (:505, ProjectionContext). Returns PSDPROJ_OK or a
 * negative error; *out is untouched on error. */
int psdproj_create(int n, const psdproj_params* p, void* ws, size_t ws_bytes, psdproj_ctx* out);

/* Project A (device, n x n, lda) into Pi (device, ldpi). tol: absolute per-pair residual
 * 2-norm threshold. info may be NULL. */
int psdproj_project(psdproj_ctx ctx, const double* A, int lda, double* Pi, int ldpi, double tol,
                    void* stream, psdproj_info* info);

/* Same, with HOST A and Pi (pinned or pageable): H2D copy of A, projection, D2H copy of Pi,
 * all on `stream` inside the call (the end-to-end path). */
int psdproj_project_host(psdproj_ctx ctx, const double* A_host, int lda, double* Pi_host, int ldpi,
                         double tol, void* stream, psdproj_info* info);

/* ---- row-sharded mode (one matrix over the GPUs of a node) ----
 * Every rank holds the contiguous row block [row0, row0 + nrows) of A (nrows x n, lda >= nrows)
 * and receives the same rows of Pi; rank r's block must start where rank r-1's ends. Per LOBPCG
 * iteration the library all-gathers the new directions W (for the block multiply A_local W),
 * all-reduces the Gram partials and column sums of squares (NCCL, on the call's stream), and
 * runs the small dense Rayleigh-Ritz step replicated (identical inputs -> identical decisions on
 * every rank). Pi_local = W_local W^T (W = V diag(sqrt(theta+)), gathered). The exact
 * eigensolver (DIRECT) is not available: such calls return PSDPROJ_E_CAPACITY.
 * NCCL is loaded at run time (dlopen libnccl.so.2 or PSDPROJ_NCCL_LIB). */
int psdproj_get_nccl_uid(void* uid_out /* 128 bytes, host */);
size_t psdproj_workspace_bytes_sharded(int n, int nrows_max, int nranks, const psdproj_params* p);
int psdproj_create_sharded(int n, int row0, int nrows, const void* nccl_uid, int rank, int nranks,
                           const psdproj_params* p, void* ws, size_t ws_bytes, psdproj_ctx* out);

/* Batched: count independent contexts (one per cone block, possibly different n). The blocks are
 * driven by up to PSDPROJ_BATCH_THREADS (env, default 8) host threads, each on its own stream
 * forked from and joined back to `stream` (the latency-bound iterations of different blocks
 * overlap on the GPU). Distinct ctxs are required. Per-item status in infos[i].status; returns
 * the worst status (or the first negative error code). */
int psdproj_project_batched(psdproj_ctx* ctxs, int count, const double* const* A, const int* lda,
                            double* const* Pi, const int* ldpi, const double* tol, void* stream,
                            psdproj_info* infos);

/* f4: many tiny cone blocks (n_i <= 112) in one launch, one CTA per block: the exact
 * projection by the one-CTA Jacobi eigensolver in shared memory, Pi_i = sum_{lambda > 0} lambda v v^T
 * (or A_i - sum_{lambda < 0}, whichever side has fewer eigenvalues), exactly
 * symmetric. No context and no warm state (the blocks are small enough for the exact path, R50).
 * Host arrays n, A (device pointers), lda, Pi (device pointers, may equal A), ldpi of length count;
 * npos_host (host, nullable) receives the positive-eigenvalue counts. Synchronous on `stream`.
 * Errors: PSDPROJ_E_CAPACITY for n_i > 112, PSDPROJ_E_DEGENERATE if a Jacobi run does not converge. */
int psdproj_project_tiny_batched(int count, const int* n, const double* const* A, const int* lda,
                                 double* const* Pi, const int* ldpi, int* npos_host, void* stream);

/* f4 (PAPER.md:605-649 -- BO-like blocks with rank-one / low-rank PSD parts): one CTA runs
 * the whole warm-started LOBPCG (Alg. 3, positive side) of each tiny block (1 <= n_i <= 112) in shared
 * memory, one launch for the batch. Xw[i]: caller-owned device warm block (n_i x 8, ld n_i); m_state[i]
 * (host, in/out): its width (0 = cold: m0 Philox columns keyed by seed, block index and `call`). tol: the
 * per-pair residual threshold; guard: non-positive guard columns (>= 1, R8/R12).
 * Outputs (host arrays of count): status 0 OK / 1 NOT_CONVERGED (max_iter) / 3 computed by the exact
 * one-CTA path because the block outgrew 8 columns or its pencil stayed singular; iters; npos; bound
 * (Theorem 3 from an explicit B V+, R53; 0 for status 3). Pi[i] (device) is exactly symmetric. ws: device
 * scratch of psdproj_tiny_lobpcg_ws_bytes(count), 16-byte aligned. Synchronous on stream. */
size_t psdproj_tiny_lobpcg_ws_bytes(int count);
int psdproj_project_tiny_lobpcg(int count, const int* n, const double* const* A, const int* lda, double* const* Pi,
                                const int* ldpi, double* const* Xw, int* m_state, double tol, int max_iter, int guard,
                                int m0, uint64_t seed, uint32_t call, void* ws, size_t ws_bytes, int* status,
                                int* iters, int* npos, double* bound, void* stream);

/* Warm block of the last call (the warm start the next call uses): vals_host (cap
 * values, descending Ritz values of the side used, sign as computed on B = side*A), vecs_dev (n x cap,
 * ldv, device, caller-owned) may be NULL. Returns the count (>= 0) or a negative error. */
int psdproj_get_ritz(psdproj_ctx ctx, double* vals_host, int cap, double* vecs_dev, int ldv);

/* Drop the warm state (`warm` optional): the next call is cold -- Philox start block,
 * side hint / positive side (PAPER.md:505 needs the previous counts). Returns PSDPROJ_OK or < 0. */
int psdproj_reset(psdproj_ctx ctx);

/* Free the host-side context and the streams / events it created (never the caller's workspace).
 * Returns PSDPROJ_OK, or PSDPROJ_E_INVALID for NULL. */
int psdproj_destroy(psdproj_ctx ctx);

/* Thread-local message of the last error ("" if none). */
const char* psdproj_last_error(void);

/* ---- f1/f3: approximate ADMM (Alg. 1) for diagonal SDPs (MaxCut: BASELINE configs[4]) ----
 * min <Q, X> s.t. X_ii = b_i for the i with w_i = 1, X in S+, as A x = z, z in C = {b}^w x S+ with
 * A = [D_w; I], P = 0. b, w: device vectors of length n, or NULL for b = 1, w = 1 (MaxCut).
 * step1: the elementwise KKT solve of line 3 (A^T A is diagonal), the relaxation of line 4, and the
 * projection input V = alpha X~ + (1 - alpha) Zp + Yp / rho of line 5 (Zh = the relaxed z-hat,
 * zeh its diagonal part). The caller projects V with psdproj_project (Zp <- Pi(V), tolerance
 * 10/k^1.01). step2: the dual update of line 6 and the residual maxima
 * res_host[0..2] = (max|X - Zp|, max_{w_i=1} |X_ii - b_i|, max|Q + Yp + Diag(w ye)|) (host,
 * synchronous). All matrices n x n, column-major, ld, device; ye, zeh length n, device. The
 * successive differences of (X, ye, Yp) are the infeasibility certificates of Theorem 1 (PAPER.md:100-119,
 * f3, checked by the caller). Reading R43. */
int psdproj_admm_maxcut_step1(int n, double* X, const double* Zp, const double* Yp, const double* ye,
                              const double* Q, int ld, double sigma, double rho, double alpha, double* Zh,
                              double* V, double* zeh, const double* b, const double* w, void* stream);
int psdproj_admm_maxcut_step2(int n, const double* X, const double* Zp, const double* Zh, double* Yp, double* ye,
                              const double* zeh, const double* Q, int ld, double rho, double* res_host,
                              const double* b, const double* w, void* stream);

/* f3 (Theorem 1; practical tests PAPER.md:563-587, reading R49): the certificate
 * terms of two successive iterates (X, ye, Yp) and (X0, ye0, Yp0) of the diagonal-SDP ADMM above, in
 * one pass on the device: terms_host[0..6] (host) = ||dX||_F^2, ||w dye||^2, ||dYp||_F^2, b.(w dye),
 * <Q, dX>, ||w diag dX||^2, max|dYp + Diag(w dye)| (d = difference). Also writes dY_sym = sym(dYp) and
 * mdX_sym = -sym(dX) (n x n, ld, device), whose PSD parts the caller takes with psdproj_project
 * (DIRECT). work: device scratch of work_elems doubles (>= 7 (2 SMs + 1)). Synchronous on stream. */
int psdproj_admm_certificate_terms(int n, const double* X, const double* X0, const double* ye, const double* ye0,
                                   const double* Yp, const double* Yp0, const double* Q, int ld, const double* b,
                                   const double* w, double* dY_sym, double* mdX_sym, double* work, size_t work_elems,
                                   double* terms_host, void* stream);

/* ---- kernel-level entry points (tests and benchmarks call the same kernels the path uses) ---- */

/* C = alpha op(A) op(B) + beta C, column-major, opA/opB: 0 = N, 1 = T. ws: device scratch of
 * ws_elems doubles for split-K partials (may be NULL). Device pointers. */
int psdproj_dgemm(int opA, int opB, int M, int N, int K, double alpha, const double* A, int lda,
                  const double* B, int ldb, double beta, double* C, int ldc, double* ws,
                  size_t ws_elems, void* stream);

/* The a3 block multiply exactly as the path runs it: Y = alpha A Z with A symmetric
 * (n x n, lda even, 16-byte aligned), Z (n x k, ldz even), Y (n x k, ldy); TMA-staged 128-byte-swizzled
 * tiles + DMMA (gemm_tma.cuh). ws: split-K partials (NULL = no split). Device pointers, async. */
int psdproj_symm_multiply(int n, int k, double alpha, const double* A, int lda, const double* Z, int ldz, double* Y,
                          int ldy, double* ws, size_t ws_elems, void* stream);

/* Symmetric eigendecomposition by parallel-order Jacobi (a7/a13): A (s x s, device) ->
 * w (s, ascending, device) and V (s x s, ldv, device). ws: device scratch of
 * psdproj_jacobi_ws_elems(s) doubles. Returns sweeps (>0) or a negative code. */
size_t psdproj_jacobi_ws_elems(int s);
int psdproj_jacobi(int s, const double* A, int lda, double* w, double* V, int ldv, double* ws,
                   void* stream);

/* Top-m eigenpairs of a symmetric s x s matrix by the path's Rayleigh-Ritz eigensolver (a7):
 * Householder tridiagonalisation, bisection, inverse iteration, back-transformation.
 * w (m, device, DESCENDING), V (s x m, ldv, device), npos (device int: #eigenvalues > 0).
 * ws: device scratch of psdproj_eigh_ws_elems(s, m) doubles. */
size_t psdproj_eigh_ws_elems(int s, int m);
int psdproj_eigh(int s, const double* A, int lda, int m, double* w, double* V, int ldv, int* npos,
                 double* ws, void* stream);

/* In-place Cholesky G = L L^T of the path's implicit Cholesky-QR (a6): G (t x t,
 * ld, device) -> lower triangle L, upper triangle zeroed. Returns 0, or j + 1 when pivot j is
 * <= 1e-12 * max diag(G) (R20; G is then left partially factored), or a negative error code. */
int psdproj_cholesky(int t, double* G, int ld, void* stream);

/* Raw Philox4x32-10 stream: out[4i+j] for counters (i, c1, c2, c3), key (k0, k1), device out. */
int psdproj_philox_raw(int count, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                       uint32_t* out, void* stream);

/* n x q N(0,1) block with the expansion mapping of R11 (device out, ld). */
int psdproj_philox_gauss(int n, int q, double* out, int ld, uint64_t seed, uint32_t stream_id,
                         uint32_t ctx, uint32_t tag, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PSDPROJ_H */
