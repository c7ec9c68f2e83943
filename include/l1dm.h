/*
 * l1dm.h — C ABI of the B200-native l1 distance-matrix block product.
 *
 *   Y = A·Z,   A_ij = ||x_i - x_j||_1 = sum_k |x_ik - x_jk|      (§2)
 *
 * computed without forming A, by the paper's method: a one-time per-coordinate
 * sort (Alg. 1) and, per query, prefix sums in sorted order plus one
 * rank lookup per point and coordinate (Alg. 2; Thm "p=1").
 * A block Z of m columns is m independent matvecs (Lemma matrixmult).
 *
 * Every entry point returns a status code; nothing crosses the ABI as an
 * exception or abort.  A thread-local message for the last failure is available
 * from l1dm_last_error().  There is no CPU fallback: without a usable sm_100
 * device every call that needs one returns L1DM_EDEVICE.
 *
 * Pointers may be HOST or DEVICE memory unless a parameter says otherwise; the
 * library classifies each with cudaPointerGetAttributes.  Host buffers are
 * staged through library-owned device buffers.  Pageable host buffers make the call
 * synchronous.  A query whose Z and Y are both PINNED host memory (cudaHostAlloc /
 * cudaHostRegister) is asynchronous like a device-pointer call: its H2D and D2H copies run
 * on the handle's copy streams through two staging slots, so consecutive queries overlap
 * their copies with each other's compute; call l1dm_sync before reading Y or reusing Z.
 *
 * Layouts (all row-major, C order):
 *   X  n x ld_x  fp32  (point i at X + i*ld_x; coordinates k_begin..k_end-1 used)
 *   Z  n x ld_z  fp32  (query column c of point j at Z[j*ld_z + c], c < m)
 *   Y  n x ld_y  fp64  (output, OVERWRITTEN, never accumulated into)
 *
 * Threads / streams: a handle is bound to the CUDA device current when it was
 * prepared.  Calls on one handle must be serialised by the caller (its query
 * workspace is shared); use one handle per concurrent stream.  Prepared state
 * is immutable after l1dm_prepare returns, so handles may be queried from
 * several streams only if each has its own handle.
 */
#ifndef L1DM_H
#define L1DM_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define L1DM_API __attribute__((visibility("default")))
#else
#define L1DM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct l1dm_ctx *l1dm_handle; /* opaque; owns every internal device buffer */

typedef enum {
  L1DM_OK = 0,
  L1DM_EINVAL = -1,     /* null pointer, n/d/m < 1, n >= 2^32, bad leading dimension or range */
  L1DM_ENONFINITE = -2, /* X holds a NaN or +-Inf (point sets are finite) */
  L1DM_ENOMEM = -3,     /* a device or pinned-host allocation failed */
  L1DM_ECUDA = -4,      /* a CUDA runtime error (message in l1dm_last_error) */
  L1DM_EDEVICE = -5,    /* no sm_100 device, or the handle belongs to another device */
  L1DM_ENOTIMPL = -6,
  L1DM_ETIMEOUT = -7,   /* a look-back wait exceeded its bound (never expected; results invalid) */
  L1DM_ENOTSIMPLEX = -8 /* TV query on rows that are not probability vectors (Thm. tv) */
} l1dm_status;

/* ---------------------------------------------------------------------------
 * Prepare — Alg. 1: for every coordinate k, a stable ascending
 * sort of x_{.k}, kept as
 *   sval[k][r] = x_{perm[k][r], k}   sorted values T_k
 *   perm[k][r]                       the order pi^k induced by T_k
 *   rank[k][i] = r with perm[k][r]=i "position of x_i(k) in T_k"
 *                (built on the handle's stream by the first query that reads it — gather
 *                mode — not by prepare: scatter and runs queries never need it)
 *   h[i]       = sum_k x_ik (fp64)   per-point coordinate sum (query epilogue)
 * plus, when every coordinate takes <= 256 distinct values, the runs tables.
 * Ties are ordered by point index; -0.0 is ordered as +0.0.
 * X: n x d fp32 (ld_x = d), host or device, BORROWED for the call only (the
 * library copies what it needs).  Synchronous: returns when the state is
 * complete.  Errors: EINVAL (X or out null, n < 1, d < 1, n >= 2^32),
 * ENONFINITE, ENOMEM, ECUDA, EDEVICE.  On error *out is set to NULL.
 * ------------------------------------------------------------------------- */
L1DM_API l1dm_status l1dm_prepare(const float *X, int64_t n, int64_t d, l1dm_handle *out);

/* Coordinate shard: prepare only coordinates [k_begin, k_end) of X (n x ld_x).
 * Queries on the handle then return the shard's PARTIAL product
 *   Y_g = sum_{k in [k_begin,k_end)} A^(k) Z,  A^(k)_ij = |x_ik - x_jk|,
 * including the shard's own share of the epilogue, so that the sum of Y_g over
 * a partition of [0, d) is A·Z exactly up to rounding (swap of sums).
 * `stream` (a cudaStream_t; NULL = the legacy default stream, CUDA's convention) is
 * used for the prepare work and becomes the handle's stream (used by l1dm_matvec,
 * l1dm_sync, l1dm_free).  Synchronous. */
L1DM_API l1dm_status l1dm_prepare_ex(const float *X, int64_t n, int64_t ld_x, int64_t k_begin,
                            int64_t k_end, void *stream, l1dm_handle *out);

/* ---------------------------------------------------------------------------
 * Query — Alg. 2 for the m columns of Z at once:
 *   y_i = sum_k [ x_ik (S3 - S4) + S2 - S1 ]  per column
 * evaluated in the equivalent single-array form
 *   y_i = 2 sum_k U^k_{rank_k(i)} + g - h_i S,  U^k_r = v_r P_r - Q_r,
 * P, Q the exclusive prefix sums of z and x·z in sorted order, S = 1^T Z,
 * g = h^T Z; fp64 accumulation of the fp32 inputs.
 * Z: n x m fp32 (ld_z = m); Y: n x m fp64 (ld_y = m), OVERWRITTEN.
 * Device Z/Y: stream-ordered on the handle's (prepare) stream; Z and Y must stay valid
 * until the stream reaches the end of the call.  Host Z/Y: synchronous.
 * NaN/Inf in Z are not checked; they propagate into Y by IEEE rules (in the fixed-point scatter
 * mode: a column of Z holding a NaN or Inf gives a NaN column of Y).
 * Errors: EINVAL (null, m < 1), EDEVICE, ENOMEM (workspace), ECUDA. */
L1DM_API l1dm_status l1dm_matvec(l1dm_handle h, const float *Z, int64_t m, double *Y);

/* As l1dm_matvec with explicit leading dimensions (ld_z >= m, ld_y >= m) and
 * stream (NULL = the legacy default stream, CUDA's convention).  The work is
 * ordered on that stream only: Z must be ready on it, Y is ready when it is. */
L1DM_API l1dm_status l1dm_matvec_ex(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m, double *Y,
                           int64_t ld_y, void *stream);

/* As l1dm_matvec_ex (device Z and Y only), for overlapping the cross-GPU sum of Y with the
 * query: the pass that completes Y (the last accumulate) runs per contiguous point block
 * b = 0..point_blocks-1 (rows [floor(b n / B), floor((b+1) n / B))), and block_events[b]
 * (a cudaEvent_t created by the caller; NULL entries are skipped) is recorded on `stream`
 * right after block b's rows of Y are final.  Errors as l1dm_matvec_ex, and EINVAL for
 * point_blocks < 1 or > n. */
L1DM_API l1dm_status l1dm_matvec_pipelined(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                           double *Y, int64_t ld_y, void *stream,
                                           int64_t point_blocks, void *const *block_events);

/* ---------------------------------------------------------------------------
 * l_p^p for odd p (Thm. odd_p: "O(nd log n) preprocessing and
 * O(ndp) query"; the paper omits the construction, SPEC S:150-158 gives it):
 *   Y = A_p Z,  (A_p)_ij = ||x_i - x_j||_p^p = sum_k |x_ik - x_jk|^p,  p in {1, 3, 5, 7}.
 * Same prepared state as l1dm_matvec (the sort of Alg. 1).  Per coordinate the query carries
 * the p+1 prefix moments M_t(r) = sum_{r'<r} z_{perm(r')} v_{r'}^t in sorted order, and
 *   y_i += sum_t C(p,t) (-1)^t x_ik^(p-t) (2 M_t(rank_k(i)) - M_t(n))
 * (|a - b|^p = sign(a - b)(a - b)^p for odd p, binomial expansion).  p = 1 is l1dm_matvec.
 * fp64 throughout; the moments of large |x| lose relative accuracy with p (R18).
 * Layouts, streams, host/device pointers and errors as l1dm_matvec_ex, plus EINVAL for p not
 * in {1, 3, 5, 7}.  Sharded handles return the shard's partial product. */
L1DM_API l1dm_status l1dm_matvec_lp_ex(l1dm_handle h, int p, const float *Z, int64_t ld_z,
                                       int64_t m, double *Y, int64_t ld_y, void *stream);
L1DM_API l1dm_status l1dm_matvec_lp(l1dm_handle h, int p, const float *Z, int64_t m, double *Y);

/* ---------------------------------------------------------------------------
 * Total variation (Thm. tv: "follows immediately from our l1 result"):
 *   Y = A_TV Z,  (A_TV)_ij = TV(x_i, x_j) = ||x_i - x_j||_1 / 2,
 * for rows x_i on the probability simplex.  The first TV call on a handle checks
 * the prepared data once (one small reduction and a synchronisation): every coordinate >= 0 and,
 * when the handle holds whole rows (k_begin = 0, k_end = ld_x), |sum_k x_ik - 1| <= 1e-9 +
 * d 2^-23 (fp32 rounding of the entries, R17); otherwise ENOTSIMPLEX.  A coordinate
 * shard can only check non-negativity: the caller owns the row-sum check across shards.
 * Layouts, streams, pointers and other errors as l1dm_matvec_ex. */
L1DM_API l1dm_status l1dm_tv_matvec_ex(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                       double *Y, int64_t ld_y, void *stream);
L1DM_API l1dm_status l1dm_tv_matvec(l1dm_handle h, const float *Z, int64_t m, double *Y);

/* ---------------------------------------------------------------------------
 * Sort-free l_p^p for even p (Alg. "query_p_even" and Thm. even_p,
 * P:453-481, with the C(p,t) and y_j the text drops — SPEC S:140-146, R19; p = 2
 * is the squared-Euclidean case of Alg. 3):
 *   Y = A_p Z,  (A_p)_ij = sum_k (x_ik - x_jk)^p,  p in {2, 4, 6},
 *   y_ic = sum_k sum_t C(p,t) (-1)^t x_ik^(p-t) W_t[k][c],  W_t[k][c] = sum_j x_jk^t z_jc.
 * No preprocessing and no handle: X (n x ld_x fp32, d coordinates used), Z (n x ld_z fp32),
 * Y (n x ld_y fp64, OVERWRITTEN).  Device pointers: stream-ordered on `stream` (scratch from
 * the stream-ordered allocator); any host pointer makes the call synchronous (staged).
 * fp64 accumulation of fp32 inputs; the moments of large |x| cancel (R18).
 * Errors: EINVAL (null, sizes, leading dimensions, p not in {2, 4, 6}), EDEVICE, ENOMEM,
 * ECUDA. */
L1DM_API l1dm_status l1dm_lpp_even_matvec(const float *X, int64_t n, int64_t ld_x, int64_t d,
                                          int p, const float *Z, int64_t ld_z, int64_t m,
                                          double *Y, int64_t ld_y, void *stream);

/* The bilinear form of Thm. maha (the paper's "Mahalanobis distance squared" is
 * f(x, y) = x^T M y for a d x d matrix M, R20):
 *   Y = A Z,  A_ij = x_i^T M x_j,  i.e. Y = X (M (X^T Z))   (Alg. 8: v = S y, z(k) = <x_k, v>,
 * with Alg. 7's S = M X^T applied, not stored).  M: d x d fp64 row-major (host or device).
 * No handle; pointers, streams and errors as l1dm_lpp_even_matvec (EINVAL for a NULL M). */
L1DM_API l1dm_status l1dm_bilinear_matvec(const float *X, int64_t n, int64_t ld_x, int64_t d,
                                          const double *M, const float *Z, int64_t ld_z, int64_t m,
                                          double *Y, int64_t ld_y, void *stream);

/* ---------------------------------------------------------------------------
 * Approximate l2 through the l1 engine (Thm. l2embed P:623-631,
 * Algs. "Preprocessing" for l2 and Thm. l2_approx):
 *   Xp[i][r] = (1 / (beta k)) sum_j G[r][j] X[i][j],   beta = sqrt(2/pi),   r < k,
 * G a k x d matrix of i.i.d. N(0,1) draws supplied by the caller (the method's random numbers
 * are an input, R22), fp64 accumulation rounded to fp32.  Then l1dm_prepare(Xp)
 * and l1dm_matvec give B Z with B_ij = ||Xp_i - Xp_j||_1 = (1 +- eps) ||x_i - x_j||_2 w.h.p.
 * for k = O(log n / eps^2).  Device pointers only (X: n x ld_x, G: k x d dense, Xp: n x ld_p);
 * stream-ordered.  Errors: EINVAL (null, sizes, host pointers), EDEVICE, ECUDA. */
L1DM_API l1dm_status l1dm_l2_embed(const float *X, int64_t n, int64_t ld_x, int64_t d,
                                   const float *G, int64_t k, float *Xp, int64_t ld_p,
                                   void *stream);

/* Column-block output for overlapping the cross-GPU sum in the scatter strategy, whose rows
 * are final only after the last column block: the query writes Yb, a
 * column-block-major array of col_blocks blocks of n x mb fp64 (block cb holds columns
 * [cb mb, min(m, cb mb + mb)) of Y with rows contiguous; a ragged last block is padded to mb),
 * and records block_events[cb] (caller-created cudaEvent_t; NULL entries skipped) on `stream`
 * as soon as block cb is final, so a collective on block cb can run while later blocks are
 * computed.  l1dm_query_layout reports the handle's strategy, mb and col_blocks for m (host
 * only); l1dm_unblock converts Yb back to a row-major Y (n x ld_y).  Device pointers only.
 * Errors: EINVAL (not the scatter strategy for this m, m < 2, nevents not 0 or col_blocks,
 * host pointers), and as l1dm_matvec_ex. */
L1DM_API l1dm_status l1dm_query_layout(l1dm_handle h, int64_t m, int64_t *scatter, int64_t *mb,
                                       int64_t *col_blocks);
/* The strategy an m-column l1 query on h runs (the planner's choice under the handle's mode):
 * gather (U + rank gather, HBM-bound), scatter (L2 reductions into a resident output block) or
 * runs (tie-heavy data).  Errors: EINVAL. */
#define L1DM_STRATEGY_GATHER 0
#define L1DM_STRATEGY_SCATTER 1
#define L1DM_STRATEGY_RUNS 2
L1DM_API l1dm_status l1dm_query_strategy(l1dm_handle h, int64_t m, int *strategy);
L1DM_API l1dm_status l1dm_matvec_colblocks(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                           double *Yb, void *stream, int64_t nevents,
                                           void *const *block_events);
L1DM_API l1dm_status l1dm_unblock(const double *Yb, int64_t n, int64_t m, int64_t mb, double *Y,
                                  int64_t ld_y, void *stream);

/* ---------------------------------------------------------------------------
 * Cross-GPU sum over peer memory.  The
 * coordinate shards' partials add up to Y because A = sum_k A^(k).  One
 * process per GPU; rows are owned in contiguous blocks (owner o: rows
 * [floor(o n / G), floor((o+1) n / G))).  Buffers every rank allocates with
 * l1dm_ipc_alloc and maps on every other rank with l1dm_ipc_open (handles
 * exchanged by the caller, e.g. torch.distributed):
 *   inbox  2 halves (epoch parity) of G slots of rows_o x m fp64 each (slot g of
 *          epoch e at inbox + ((e & 1) G + g) rows_o m, row stride m)
 *   flags  2G unsigned words, zero-initialised (arrivals [0, G), results [G, 2G))
 *   ybuf   n x m fp64 result (row stride m), on ranks that receive the sum
 * and one local device word for timeouts.  epoch: the caller's query counter,
 * strictly increasing from 1 (a wait ends when a flag reaches at least it).
 * Stream order per rank: l1dm_matvec_push, l1dm_peer_reduce, then (result ranks)
 * l1dm_peer_wait; l1dm_peer_check reports a timed-out wait (the result is
 * then invalid).  These calls wait on other GPUs' kernels: never run several
 * ranks of one group on one GPU (nothing guarantees those kernels co-run); a
 * single-GPU emulation must issue every rank's push before any reduce. */
#define L1DM_MAX_PEERS 16
typedef struct {
  int world;                        /* G, 1..L1DM_MAX_PEERS */
  int rank;                         /* this rank */
  double *inbox[L1DM_MAX_PEERS];    /* owner o's inbox as mapped in this process */
  unsigned *flags[L1DM_MAX_PEERS];  /* owner o's 2G flag words as mapped here */
  double *ybuf[L1DM_MAX_PEERS];     /* rank t's result buffer as mapped here, or NULL */
  unsigned *timeout;                /* this rank's timeout word (device, zeroed) */
  int64_t n;                        /* points and columns the inboxes and result buffers were */
  int64_t m;                        /* allocated for: every call checks its n, m against them */
} l1dm_peer_t;
/* bytes of device memory, zeroed, with its 64-byte CUDA IPC handle in handle[0..64). */
L1DM_API l1dm_status l1dm_ipc_alloc(size_t bytes, void **dptr, void *handle);
L1DM_API l1dm_status l1dm_ipc_free(void *dptr);
/* Map another process's allocation (same node; peer access enabled lazily). */
L1DM_API l1dm_status l1dm_ipc_open(const void *handle, void **dptr);
L1DM_API l1dm_status l1dm_ipc_close(void *dptr);
/* This rank's partial A^(K_g) Z (m columns of device Z) goes row by row into the owners'
 * inbox slots — stored by the query's final pass itself (gather mode's last accumulate,
 * scatter mode's block write-out: peer stores over NVLink that overlap the pass), or pushed
 * after a local pass (m = 1 scatter, runs) — then rank g's arrival flag is raised at every
 * owner.  Stream-ordered; Errors: EINVAL (arguments, epoch 0, unmapped peers), as
 * l1dm_matvec_ex. */
L1DM_API l1dm_status l1dm_matvec_push(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                      const l1dm_peer_t *peers, unsigned epoch, void *stream);
/* Owner side (every rank): wait for the G arrivals of this epoch, sum the G slots of this
 * rank's rows in rank order (deterministic) and store them into ybuf[t] of every rank t whose
 * bit is set in targets (the root for a reduce, all ranks for an all-reduce), then raise this
 * owner's result flag at each target. */
L1DM_API l1dm_status l1dm_peer_reduce(const l1dm_peer_t *peers, int64_t n, int64_t m,
                                      unsigned epoch, unsigned targets, void *stream);
/* Result side: wait for every owner's rows of this epoch; then, if Y is not NULL, copy the
 * n x m result from this rank's ybuf into Y (device, row stride ld_y). */
L1DM_API l1dm_status l1dm_peer_wait(const l1dm_peer_t *peers, unsigned epoch, int64_t n, int64_t m,
                                    double *Y, int64_t ld_y, void *stream);
/* Synchronise the stream and report (then clear) a timed-out peer wait: ETIMEOUT.  After a
 * timeout the epoch-parity reuse argument no longer holds: tear the group down and allocate a
 * fresh one (the Python PeerGroup does this) rather than continuing with the next epoch.
 * A timed-out wait ends every other wait of the same rank early (they poll the timeout word). */
L1DM_API l1dm_status l1dm_peer_check(const l1dm_peer_t *peers, void *stream);

/* ---------------------------------------------------------------------------
 * Matrix-free consumers of the block product (PAPER.md "Applications",
 * P:727-817): everything between the products runs in this library too (fp64 tensor-core
 * GEMMs, a device Jacobi eigensolver, device-scalar conjugate gradients); DESIGN.md §2d.
 *
 * An operator names the matrix A the consumers touch only through products A V:
 *   L1DM_OP_SORTED    a prepared handle h, p in {1, 3, 5, 7}: A_ij = ||x_i - x_j||_p^p
 *                     (l1dm_matvec / l1dm_matvec_lp; n = the handle's points)
 *   L1DM_OP_EVEN      X (n x ld_x fp32, d coordinates, device), p in {2, 4, 6}:
 *                     A_ij = ||x_i - x_j||_p^p sort-free (l1dm_lpp_even_matvec)
 *   L1DM_OP_BILINEAR  X as above and M (d x d fp64, device): A_ij = x_i^T M x_j
 *                     (l1dm_bilinear_matvec; PSD when M is, the CG case of Thm. linear_system)
 * The products take fp32 blocks (BASELINE.json); an fp64 block V is applied as
 * A fp32(V) + A fp32(V - fp32(V)) in one product of width 2b (linearity, R21).
 * Every buffer below is DEVICE memory; every call is stream-ordered on `stream` unless it says
 * otherwise, and uses the stream-ordered allocator for its scratch. */
#define L1DM_OP_SORTED 0
#define L1DM_OP_EVEN 1
#define L1DM_OP_BILINEAR 2
typedef struct {
  int kind;            /* L1DM_OP_* */
  int p;               /* exponent (SORTED: 1, 3, 5, 7; EVEN: 2, 4, 6; BILINEAR: ignored) */
  l1dm_handle h;       /* SORTED */
  const float *X;      /* EVEN, BILINEAR: n x ld_x fp32 */
  int64_t n, ld_x, d;  /* EVEN, BILINEAR (SORTED: n is taken from the handle) */
  const double *M;     /* BILINEAR: d x d fp64 row-major */
} l1dm_operator_t;

/* C (M x N, ldc) = alpha op(A) B + beta C in fp64 on the tensor cores (DMMA), deterministic:
 *   trans_a = 0: op(A) = A, A is M x K (lda);  trans_a = 1: op(A) = A^T, A is K x M (lda);
 *   B is K x N (ldb); all row-major.  beta = 0 never reads C.  Errors: EINVAL (null, sizes,
 *   leading dimensions), EDEVICE, ENOMEM, ECUDA. */
L1DM_API l1dm_status l1dm_gemm(int trans_a, int64_t M, int64_t N, int64_t K, double alpha,
                               const double *A, int64_t lda, const double *B, int64_t ldb,
                               double beta, double *C, int64_t ldc, void *stream);

/* Symmetric eigen-decomposition by cyclic Jacobi (round-robin parallel ordering): A (N x N,
 * lda, symmetric; only read) -> W (N eigenvalues, in no particular order) and V (N x N, ldv;
 * column j is the unit eigenvector of W[j]).  Errors: EINVAL, EDEVICE, ENOMEM, ECUDA. */
L1DM_API l1dm_status l1dm_syevj(int64_t N, const double *A, int64_t lda, double *W, double *V,
                                int64_t ldv, void *stream);

/* The k eigenpairs of largest |lambda| of a symmetric A (N x N, lda; only read): Householder
 * tridiagonalisation on a cooperative grid, Sturm bisection, inverse iteration with
 * re-orthogonalisation inside eigenvalue clusters, back-transformation.  lam[k] in
 * nonincreasing |lambda| order (ties: smaller eigenvalue index first), V (N x k, ldv) the unit
 * eigenvectors.  N <= 4096, k <= min(N, 96).  Errors: EINVAL, EDEVICE, ENOMEM, ECUDA. */
L1DM_API l1dm_status l1dm_syev_topk(int64_t N, const double *A, int64_t lda, int64_t k,
                                    double *lam, double *V, int64_t ldv, void *stream);

/* Y (n x b, ldy) = A V for an fp64 block V (n x b, ldv) through the operator's fp32 product
 * (hi/lo split, one product of 2b columns).  Errors: EINVAL (operator, sizes), as the
 * operator's product. */
L1DM_API l1dm_status l1dm_op_apply(const l1dm_operator_t *op, const double *V, int64_t ldv,
                                   int64_t b, double *Y, int64_t ldy, void *stream);

/* Randomized block Krylov for the k largest |eigenvalues| of the symmetric A = its top-k
 * singular values (Thm. musco; Thm. bakshi22 P:727-731 via Thm. opt_lowrank_p
 * P:757-766): K = [A Pi, A^2 Pi, ..., A^q Pi], each new block orthonormalised
 * against the earlier ones (block classical Gram-Schmidt: against the last two blocks, then
 * against the whole basis) and within itself (CholeskyQR2 with column dropping: columns whose
 * residual is below 1e-7 of the block's largest column norm are dropped as zero columns: the
 * Krylov space is exhausted), the Rayleigh quotient T = Q^T A Q
 * assembled from the orthogonalisation coefficients (block Lanczos with full
 * re-orthogonalisation), its k eigenpairs of largest |lambda| (as l1dm_syev_topk), sigma = |lam|
 * in nonincreasing order, Z = Q V_k.  q + 1 block products of width 2b.
 * Pi: the n x b start block (the method's random draw; the caller passes it, e.g. i.i.d.
 * N(0,1) from a seeded generator).  1 <= k <= b <= 96, q >= 1, q b <= min(n, 4096).
 * Outputs: sigma[k], lam[k] (signed Ritz values), Z (n x k, ldz, orthonormal columns); any
 * output may be NULL except sigma.  Synchronous (returns when the outputs are ready).
 * Errors: EINVAL, as l1dm_op_apply, ENOMEM, ECUDA. */
typedef struct {
  int64_t products;   /* block products A V */
  int64_t columns;    /* fp32 columns through the product (2b per product) */
  int64_t block, depth;
  double product_ms;  /* device time in the products (CUDA events on `stream`) */
  double total_ms;    /* device time of the whole call */
} l1dm_krylov_info_t;
L1DM_API l1dm_status l1dm_block_krylov(const l1dm_operator_t *op, int64_t k, int64_t block,
                                       int64_t depth, const double *Pi, double *sigma,
                                       double *lam, double *Z, int64_t ldz, void *stream,
                                       l1dm_krylov_info_t *info);

/* The same with a caller-supplied product instead of an operator, e.g. a coordinate-sharded
 * partial product followed by the cross-GPU all-reduce (A = sum_g A^(K_g)): every dense
 * step still runs in this library, identically on every rank (deterministic kernels), and only
 * the products go through the callback.  apply(user, V, ldv, b, Y, ldy, stream) must enqueue
 * Y (n x b fp64, ldy) = A V (n x b fp64, ldv) on `stream` (device pointers) and return 0 (a
 * negative l1dm_status otherwise, passed through).  Errors: as l1dm_block_krylov. */
typedef int (*l1dm_apply_fn)(void *user, const double *V, int64_t ldv, int64_t b, double *Y,
                             int64_t ldy, void *stream);
L1DM_API l1dm_status l1dm_block_krylov_cb(int64_t n, l1dm_apply_fn apply, void *user, int64_t k,
                                          int64_t block, int64_t depth, const double *Pi,
                                          double *sigma, double *lam, double *Z, int64_t ldz,
                                          void *stream, l1dm_krylov_info_t *info);

/* Conjugate gradients for A x = b (Thm. linear_system) with every scalar on the
 * device: the host only looks at the convergence flag every 8 iterations (asynchronous copy,
 * one chunk in flight), iterations after convergence leave x unchanged.  A must be symmetric
 * positive definite; normal_equations = 1 solves A^2 x = A b instead (symmetric indefinite A,
 * such as l1 distance matrices), two products per iteration.  Stops when
 * ||r|| <= tol ||rhs|| or after maxit iterations (then converged = 0: reported, never silent,
 * SPEC S:361).  b, x: n fp64 (device).  Synchronous.
 * info: iterations, relative residual ||A x - b|| / ||b|| (one more product), converged. */
typedef struct {
  int64_t iterations;
  double residual;
  int converged;
  int64_t products;
} l1dm_cg_info_t;
L1DM_API l1dm_status l1dm_cg(const l1dm_operator_t *op, const double *b, double *x, double tol,
                             int64_t maxit, int normal_equations, void *stream,
                             l1dm_cg_info_t *info);
/* CG with a caller-supplied product (see l1dm_block_krylov_cb; b = 1 column per call). */
L1DM_API l1dm_status l1dm_cg_cb(int64_t n, l1dm_apply_fn apply, void *user, const double *b,
                                double *x, double tol, int64_t maxit, int normal_equations,
                                void *stream, l1dm_cg_info_t *info);

/* Release every buffer the handle owns.  NULL is a no-op.  Synchronises the
 * handle's stream first. */
L1DM_API void l1dm_free(l1dm_handle h);

/* Wait for the handle's stream and report deferred errors: ECUDA for an
 * asynchronous fault, ETIMEOUT if a look-back wait of an earlier call gave up
 * (its Y is then invalid).  Stream-ordered device calls return before their
 * kernels finish, so this is where such failures surface. */
L1DM_API l1dm_status l1dm_sync(l1dm_handle h);

/* ---------------------------------------------------------------------------
 * Introspection and control (host-only, no compute).
 * ------------------------------------------------------------------------- */

/* Shape of a handle: points, local coordinate count, shard range. Any out may be NULL. */
L1DM_API l1dm_status l1dm_shape(l1dm_handle h, int64_t *n, int64_t *d_local, int64_t *k_begin,
                       int64_t *k_end);

/* Upper bound on the query workspace (bytes) a query with m columns allocates. */
L1DM_API size_t l1dm_workspace_bytes(l1dm_handle h, int64_t m);

/* Cap the query workspace (bytes; 0 = automatic: 75% of the free device memory).
 * A smaller cap means more coordinate chunks (more Y read-modify-writes). */
L1DM_API l1dm_status l1dm_set_workspace_limit(l1dm_handle h, size_t bytes);

/* Query strategy.  Both compute the same Y = A*Z:
 *   GATHER  the scan stores U = v*P - Q per (coordinate, sorted row) in a workspace and a
 *           per-point pass gathers U at rank_k(i) for every k (Y written once, no atomics);
 *   SCATTER one pass per column block of Y (every m, m = 1 included): the scan's tile
 *           prefixes come from a decoupled look-back over the earlier tiles of the same
 *           coordinate (Alg. 2's partial sums in sorted order; bounded waits, else
 *           ETIMEOUT) and it adds 2U straight into Y[perm_k(r)] with L2 reductions into a
 *           compact block accumulator (no U workspace, no rank gather).  Both the look-back
 *           prefixes and the accumulator are 64-bit fixed point at per-query scales bounded
 *           from Z and the sorted values, so Y is bitwise reproducible (R16); odd
 *           p > 1 accumulates in fp64 (summation order varies at the ulp level) and subtracts
 *           the coordinate totals' part with one fp64 tensor-core expansion.
 *   RUNS    tie-heavy data only (every prepared coordinate takes <= 256 distinct values,
 *           detected by prepare): Alg. 2 over the distinct values — per coordinate the run
 *           sums of Z by fp64 L2 reductions in point order, a prefix over the runs, then each
 *           point adds its run's value; no sorted-order gather at all.
 * AUTO (the default) picks RUNS when the prepared data allows it, else SCATTER when a column
 * block of Y and Z fits in L2, else GATHER.  l1_p, TV and the pipelined/column-block calls
 * follow the same choice where they apply.  Returns EINVAL for a NULL handle, an unknown
 * mode, or RUNS on data without runs tables.  Host-only. */
enum { L1DM_MODE_AUTO = 0, L1DM_MODE_GATHER = 1, L1DM_MODE_SCATTER = 2, L1DM_MODE_RUNS = 3 };
L1DM_API l1dm_status l1dm_set_query_mode(l1dm_handle h, int mode);

/* Query plan, a pure function of the sizes (testable without a GPU).
 * mb = columns per scan segment; rows_per_tile = scan tile rows; kc = coordinates
 * per chunk; chunks = ceil(d_local / kc); l2_resident = 1 when a chunk's U
 * workspace is sized to stay in L2 (small n*m); scatter = 1 when the query runs in
 * scatter mode (see l1dm_set_query_mode; mb is then the column block width). */
typedef struct {
  int64_t mb;
  int64_t col_blocks;
  int64_t vec;
  int64_t lanes_per_row;
  int64_t rows_per_tile;
  int64_t tiles_per_segment;
  int64_t kc;
  int64_t chunks;
  int64_t l2_resident;
  int64_t workspace_bytes;
  int64_t scatter;      /* 1: scatter mode, the scan adds 2U into an L2-resident Y block with reductions */
} l1dm_plan_t;
L1DM_API l1dm_status l1dm_plan(int64_t n, int64_t d_local, int64_t m, int64_t l2_bytes,
                      int64_t workspace_limit, l1dm_plan_t *out);
/* The same for an explicit query mode (L1DM_MODE_*); EINVAL for an unknown mode. */
L1DM_API l1dm_status l1dm_plan_ex(int64_t n, int64_t d_local, int64_t m, int64_t l2_bytes,
                         int64_t workspace_limit, int mode, l1dm_plan_t *out);

/* Per-kernel device time (CUDA events on the launching stream).  While enabled,
 * every launch of every kernel is bracketed by events; read accumulates the
 * durations of completed launches (it synchronises the handle's stream). */
typedef struct {
  double prep_ms;           /* l1dm_prepare total (all prepare kernels) */
  double colsums_ms;        /* K4: S = 1^T Z, g = h^T Z */
  double scan_ms;           /* K5: gather + decoupled look-back scan, writes U */
  double accumulate_ms;     /* K6: rank gather + register accumulation into Y */
  double copy_ms;           /* host<->device staging (host-pointer calls) */
  int64_t colsums_launches;
  int64_t scan_launches;
  int64_t accumulate_launches;
  int64_t queries;
  int64_t kernel_launches;  /* every kernel the library launched (prepare + queries) */
  int64_t scan_pairs;       /* (point, coordinate) pairs the timed scan launches covered */
  int64_t accumulate_pairs; /* (point, coordinate) pairs the timed accumulate launches covered */
  int64_t m_last;           /* columns of the latest query */
} l1dm_timing_t;
L1DM_API l1dm_status l1dm_timing_enable(l1dm_handle h, int enable);
L1DM_API l1dm_status l1dm_timing_read(l1dm_handle h, l1dm_timing_t *out, int reset);

/* Test-only: copy the prepared tables (each d_local x n, coordinate-major) and
 * h (n) into caller buffers (host or device; any may be NULL). */
L1DM_API l1dm_status l1dm_debug_export(l1dm_handle h, float *sval, uint32_t *perm, uint32_t *rank,
                              double *hsum);

/* Return the device blocks that freed handles left in the library's block cache (current
 * device) to CUDA.  Handles recycle each other's memory through this cache (it holds at most
 * half of the device memory and is flushed automatically when an allocation fails). */
L1DM_API l1dm_status l1dm_release_cached(void);

/* Thread-local message describing the last non-OK status ("" if none). */
L1DM_API const char *l1dm_last_error(void);

/* Kernels launched so far (this process, all devices) by the handle-free entries
 * (l1dm_lpp_even_matvec, l1dm_bilinear_matvec, l1dm_l2_embed); handle-bound launches are
 * counted per handle in l1dm_timing_t.kernel_launches.  Never fails. */
L1DM_API int64_t l1dm_handleless_launches(void);

/* Environment variables (read once per process; testing and tuning hooks — the defaults are
 * the measured choices of DESIGN.md §6 and per-handle control is l1dm_set_query_mode):
 *   L1DM_SCATTER=0|1        planner default for handles left in L1DM_MODE_AUTO (gather/scatter)
 *   L1DM_SCATTER_MB=k       scatter column-block width override
 *   L1DM_SCATTER_LB=0       scatter mode in two passes per column block (a reduce pass for
 *                           the tile totals, then the apply) instead of the look-back apply
 *   L1DM_REDUCE_ALL=0       (with L1DM_SCATTER_LB=0) tile totals by a reduce pass per block
 *   L1DM_LB_NT=128|256      threads per look-back apply CTA (tiles of 4 rows per thread)
 *   L1DM_RUNS=0             prepare never builds the runs tables (§2f)
 *   L1DM_RUNS_GATHER=0      the shared-memory-staged runs expansion
 *   L1DM_FUSED_RANK=1       the last sort pass scatters the inverse ranks eagerly
 *   L1DM_SCAN_SEGMENTS=k    gather-mode scan: split columns until k segments per chunk
 *   L1DM_K12_RING=0|1       even-p moment reduce staging variant
 *   L1DM_DEBUG_ALLOC, L1DM_DEBUG_PREP, L1DM_DEBUG_JACOBI   diagnostics to stderr
 * None changes a result beyond floating-point summation order (every path is held to the same
 * parity bar by tests/). */

/* Library version string. */
L1DM_API const char *l1dm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* L1DM_H */
