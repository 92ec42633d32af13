/*
 * hh.h -- C ABI of the B200 (sm_100a) Householder-product apply library (libhh.so).
 *
 * The operations are the apply-time computations of
 *   C. Rusu, "Approximate Eigenvalue Decompositions of Linear Transformations
 *   with a Few Householder Reflectors", arXiv:1811.07624.
 * Citations "P:L" are lines of the paper's LaTeX source (/root/reference/PAPER.md,
 * see SURVEY.md §0 for the equation/line table); the readings of ambiguous
 * passages are numbered R1..R12 in DESIGN.md.
 *
 * ----------------------------------------------------------------------------
 * Notation (Eq. 1-2; reading R1 fixes the product order):
 *   u_i = U[:, i]  (i = 1..h), U is n x h COLUMN-MAJOR with ld = n
 *         (== a row-major / C-contiguous (h, n) array, u_i contiguous)
 *   H_i = I - 2 u_i u_i^T          (Eq. 2; the stored u_i is used literally:
 *                                   no renormalisation, u_i = 0 is the identity
 *                                   slot of P:90)
 *   Q   = H_1 H_2 ... H_h
 *   X, Y, P: n x N column-major, ld = n (== C-contiguous (N, n)), column j is
 *         the contiguous n-vector at X + j*n.
 *
 * Pointers
 *   Every array pointer is a DEVICE pointer owned by the caller, except in
 *   hh_apply_host() where the data pointers are HOST pointers.  The library never
 *   allocates device memory for the caller's data, never frees or retains a
 *   pointer after the call returns, and keeps no mutable global state except a
 *   thread-safe lazily cached device-attribute table.  Scratch comes from the
 *   caller: query hh_workspace_bytes(); `workspace` may be NULL when the query
 *   returns 0.
 *
 * dtype
 *   All floating-point arrays of one call share `dtype` (HH_F32 = float,
 *   HH_F64 = double).  Index arrays are int32.
 *
 * Alignment / size
 *   - The fast kernels (fused K1 family, compact-WY tensor-core program) need every
 *     float pointer 16-byte aligned, n * sizeof(dtype) % 16 == 0 (n % 4 == 0 for f32,
 *     n % 2 == 0 for f64) and n <= 8192 (f32) / 4096 (f64).
 *   - hh_apply, hh_apply_signed, hh_apply_qr, hh_sym_apply, hh_sym_apply_signed,
 *     hh_mahalanobis, hh_congruence, hh_knn (n <= 256) and hh_apply_host take every other
 *     shape too (Eq. 1-2 hold for any n): any n >= 1 whose column fits in shared memory
 *     (n <= ~57000 f32 / ~28000 f64) and pointers aligned to the element run their
 *     reflector passes on scalar-access kernels (K1r, close to the aligned kernels'
 *     speed for n <= 4096 while U fits on chip; K1g for the rest, several times slower;
 *     hh_mahalanobis then uses its per-pair form, or with a workspace transform-once on
 *     a copy of the points at a 16-byte pitch).
 *     With the workspace hh_workspace_bytes() reports for such a shape (non-zero from the
 *     measured crossover in h), the call instead copies the operands to a 16-byte pitch,
 *     runs the fast kernels on the copy and copies the result back (two extra passes
 *     over X, flat in h).
 *     Aligned fp32 shapes with 8192 < n <= 65536 also have the tensor-core program (AUTO
 *     takes it from h = 2 on large batches when a workspace is passed).
 *   - HH_ERR_UNSUPPORTED: a pointer not aligned to its element, n beyond K1g's capacity,
 *     or HH_ALGO_WY forced on such a shape.
 *
 * Semantics
 *   - Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream); no
 *     host synchronisation except in hh_apply_host().
 *   - Y == X (exact alias) is allowed; partial overlap is undefined.
 *   - h = 0 gives Y = X (sym: Y = lambda .* X; Mahalanobis: plain weighted
 *     squared distance).  N = 0 / npairs = 0 is a successful no-op.
 *   - Arguments are validated before any launch; on error nothing is written.
 *   - Asynchronous device faults surface at the caller's next synchronising call
 *     (as in cuBLAS); HH_ERR_CUDA reports launch-time errors.
 *   - No C++ exception crosses this boundary.  All functions are thread-safe.
 *   - A workspace belongs to one call at a time: calls that may run concurrently
 *     (different streams) need distinct workspaces (as with cuBLAS workspaces).
 *   - Every call enqueues only stream-ordered work (kernels, cudaMemsetAsync): it
 *     can be captured into a CUDA graph and replayed (tests/test_graph_gpu.py).
 *   - The compact-WY projection (large h) splits a few column tiles between two CTAs
 *     of one launch: each publishes its partial in the workspace and the later of the
 *     two adds them (no CTA waits for another, so nothing assumes co-residency).
 *   - Library state: a per-device table of cached attributes (and the per-device
 *     shared-memory opt-in of its kernels); hh_set_algo and the test hooks are
 *     per calling thread.
 *
 * Preconditions NOT validated (documented): ||u_i|| = 1 or u_i = 0 for an
 * orthonormal Q; d_r >= 0; 0 <= ia[j], ib[j] < M; finite inputs.
 * ----------------------------------------------------------------------------
 */
#ifndef HH_H_
#define HH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef HH_NO_CUDA_TYPES
#include <cuda_runtime_api.h>
typedef cudaStream_t hh_stream_t;
#else
typedef void *hh_stream_t;
#endif

typedef enum {
    HH_OK = 0,
    HH_ERR_INVALID_VALUE = 1, /* bad size, NULL operand, bad op/dtype/call       */
    HH_ERR_UNSUPPORTED = 2,   /* misaligned pointer, n too big, shape a path cannot run */
    HH_ERR_WORKSPACE = 3,     /* workspace_bytes below hh_workspace_bytes()       */
    HH_ERR_CUDA = 4           /* CUDA runtime error at launch / copy              */
} hh_status;

typedef enum { HH_F32 = 0, HH_F64 = 1 } hh_dtype;

typedef enum {
    HH_OP_N = 0, /* Y = Q   X = H_1 (H_2 ( ... (H_h X)))  : u_h applied first        */
    HH_OP_T = 1  /* Y = Q^T X = H_h ( ... (H_1 X))        : u_1 applied first        */
} hh_op;
/* The paper's Eq. 1 (D = I) Ubar = U_h ... U_1 is HH_OP_T on the same
 * columns; reflector symmetry makes the transpose a reversal. */

/* Path selection for hh_apply (fp32):
 *   HH_ALGO_AUTO  -- the measured crossover: K1 fused SIMT kernel for
 *                    small h, K5 compact-WY on the tensor cores for large h when a
 *                    workspace of hh_workspace_bytes(HH_CALL_APPLY, ...) is passed; the
 *                    threshold depends on n and on the size n*N (12-19 for n >= 128 at
 *                    n*N >= 2^27, 17-26 at >= 2^25, 32 below; never K5 for n < 128);
 *   HH_ALGO_FUSED -- always K1 (any dtype);
 *   HH_ALGO_WY    -- always K5 (fp32 only; HH_ERR_WORKSPACE without a workspace,
 *                    HH_ERR_UNSUPPORTED for fp64). */
typedef enum { HH_ALGO_AUTO = 0, HH_ALGO_FUSED = 1, HH_ALGO_WY = 2 } hh_algo;

/* Side of the diagonal D of Eq. 1 (NEXT-f1, reading R2): the paper writes
 * Ubar = D U_h ... U_1 (D on the left) and Ubar_2 D in Result 3 (P:212,
 * P:237, D on the right). */
typedef enum { HH_SIDE_LEFT = 0, HH_SIDE_RIGHT = 1 } hh_side;

typedef enum {
    HH_CALL_APPLY = 0,
    HH_CALL_SYM = 1,
    HH_CALL_MAHALANOBIS = 2,
    HH_CALL_APPLY_HOST = 3,
    HH_CALL_KNN = 4,
    HH_CALL_CONGRUENCE = 5,
    HH_CALL_SHF = 6
} hh_call;

/*
 * hh_apply -- Y = Q X (op = HH_OP_N) or Y = Q^T X (op = HH_OP_T).
 *   P:42-54 (Eq. 1-2): "Matrix-vector multiplication with the matrix Ubar ...
 *   takes 4nh operations" -- each column costs h dot products u_i^T x and h
 *   rank-1 updates x -= 2 (u_i^T x) u_i, never densifying Q.
 *   n >= 1, h >= 0, N >= 0; U: n x h (may be NULL iff h == 0); X, Y: n x N.
 *   workspace: DEVICE scratch of hh_workspace_bytes(HH_CALL_APPLY, n, h, N, 0, dtype)
 *   bytes (0 when the fused kernel is selected; NULL is then fine).
 *   Small h: fused kernel K1, one HBM read + one HBM write of X (bound: HBM).
 *   Large h (fp32, workspace given): blocked compact-WY form of the same product
 *   (I - W T W^T per block of <= 256 reflectors) on the tcgen05 tensor cores with a
 *   bf16x3 split (every fp32 operand = bf16 hi + bf16 lo, products hi*hi + hi*lo + lo*hi
 *   accumulated in fp32); see hh_algo.  Same product, different rounding: the measured
 *   whole-output relative Frobenius error is 3.6e-6 / 7.3e-6 / 1.5e-5 at n = 4096,
 *   h = 64 / 256 / 1024, i.e. 10-20x the fp32 SIMT kernel's (2.5e-7 .. 1e-6)
 *   and 20-45x inside the 2e-5 sqrt(h) gate.  HH_ALGO_AUTO switches to this accuracy
 *   class at the crossover; HH_ALGO_FUSED keeps the fp32 SIMT path at any h.
 */
hh_status hh_apply(hh_op op, int64_t n, int64_t h, const void *U, const void *X,
                   void *Y, int64_t N, hh_dtype dtype, void *workspace,
                   size_t workspace_bytes, hh_stream_t stream);

/*
 * hh_sym_apply -- Y = Q diag(lambda) Q^T X.
 *   eq:thesbar with D = I (reading R2): "Matrix-vector multiplication
 *   with S-bar takes (8h+1)n operations" = a Q^T pass (u_1 first), one diagonal
 *   scale by lambda, and a Q pass (u_h first).
 *   lambda: n values of dtype (the spectrum s-bar; any sign).
 *   workspace: DEVICE scratch of hh_workspace_bytes(HH_CALL_SYM, n, h, N, 0, dtype)
 *   (0 -> fused SIMT kernel).  For fp32 and h past the measured crossover (hh_algo AUTO:
 *   7-11 for n >= 256 at n*N >= 2^27, 13-19 at >= 2^25, 32 below) the block program
 *   runs on the tensor cores: blocks 1..m-1 as Q_k^T, the last block folded with
 *   diag(lambda) into one project/update pair (Y = Lambda X - [A1 A2][G; G_lambda]),
 *   then blocks m-1..1 as Q_k.
 */
hh_status hh_sym_apply(int64_t n, int64_t h, const void *U, const void *lambda,
                       const void *X, void *Y, int64_t N, hh_dtype dtype,
                       void *workspace, size_t workspace_bytes, hh_stream_t stream);

/*
 * hh_apply_signed -- the paper's exact operator forms with the diagonal D of Eq. 1
 * (D = diag(d), d in {+-1}^n fixes det(Ubar)):
 *   side = HH_SIDE_LEFT :  Y = D op(Q) X      (Eq. 1, eq:thesbar)
 *   side = HH_SIDE_RIGHT:  Y = op(Q) D X      (Result 3)
 *   op(Q) = Q (HH_OP_N) or Q^T (HH_OP_T) as in hh_apply.  d: n values of dtype (+-1 by
 *   the paper; any diagonal is applied as given, not validated).  D is fused as a
 *   prologue/epilogue of the same kernels (n multiplies per column, no extra HBM
 *   pass).  Workspace as hh_apply.  Errors as hh_apply, plus HH_ERR_INVALID_VALUE
 *   for a bad side or a NULL d with N > 0.
 */
hh_status hh_apply_signed(hh_op op, hh_side side, int64_t n, int64_t h, const void *U,
                          const void *d, const void *X, void *Y, int64_t N, hh_dtype dtype,
                          void *workspace, size_t workspace_bytes, hh_stream_t stream);

/*
 * hh_apply_qr -- hh_apply for QR-structured ("trapezoidal") reflectors (NEXT-f2):
 *   the caller guarantees u_i[r] = 0 for r < i (0-based), the structure of the partial
 *   QR reflectors J_k of Result 3 ("k-1 leading zeros ... 4(n-k+1) operations", P:218-237,
 *   P:261; h = n-1 of them reproduce any orthonormal matrix up to +-1).  The
 *   compact-WY path (K5) skips the zero prefix -- the leading K steps of each block's
 *   projection and the leading row chunks of its update -- so a reflector costs
 *   ~4(n-i) instead of 4n (measured 1.69x at n = 4096, h = 4095); the fused small-h
 *   kernel K1 applies them in full (at small h the prefixes are a negligible share).
 *   Same arguments, workspace and errors as hh_apply; the result is identical to
 *   hh_apply on the same U when the precondition holds.
 */
hh_status hh_apply_qr(hh_op op, int64_t n, int64_t h, const void *U, const void *X, void *Y,
                      int64_t N, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                      hh_stream_t stream);

/*
 * hh_sym_apply_signed -- Y = D Q diag(lambda) Q^T D X, the symmetric form of
 * eq:thesbar with its diagonal D on both sides.  Workspace as
 * hh_sym_apply (HH_CALL_SYM).
 */
hh_status hh_sym_apply_signed(int64_t n, int64_t h, const void *U, const void *d,
                              const void *lambda, const void *X, void *Y, int64_t N,
                              hh_dtype dtype, void *workspace, size_t workspace_bytes,
                              hh_stream_t stream);

/*
 * hh_mahalanobis -- dist[j] = || D^{1/2} Q^T (P[:, ia[j]] - P[:, ib[j]]) ||^2
 *                           = (x_a - x_b)^T Q diag(d) Q^T (x_a - x_b).
 *   P:600 d_S(x_i, x_j) = ||L (x_i - x_j)||_2^2; "L = sqrt(Lambda) U ...
 *   perform the transformation x <- L x before running the k-NN" with U == Q^T
 *   (reading R4); d is the metric diagonal Lambda, d_r >= 0 (reading R3).
 *   P: n x M column-major points; ia, ib: npairs int32 indices in [0, M);
 *   dist: npairs values of dtype.
 *   workspace >= hh_workspace_bytes(HH_CALL_MAHALANOBIS, n, h, M, npairs, dtype):
 *     transform-once: Z = diag(sqrt d) Q^T P into the workspace, the pairs
 *     counting-sorted by ia on the device (histogram, scan, scatter into the
 *     workspace), then a gather kernel dist[j] = ||Z[:,ia[j]] - Z[:,ib[j]]||^2 that
 *     loads each z_a once per bucket.
 *   workspace == NULL: per-pair fused kernel (gather x_a - x_b, Q^T, weighted
 *     norm) -- no scratch, 4nh + 3n flops per pair.
 *   A non-NULL workspace smaller than the query -> HH_ERR_WORKSPACE.
 */
hh_status hh_mahalanobis(int64_t n, int64_t h, const void *U, const void *d,
                         const void *P, int64_t M, const int32_t *ia,
                         const int32_t *ib, int64_t npairs, void *dist,
                         hh_dtype dtype, void *workspace, size_t workspace_bytes,
                         hh_stream_t stream);

/*
 * hh_congruence -- M_out[b] = op(Q) M[b] op(Q)^T for `count` n x n column-major
 *   matrices (NEXT-f4): the two-sided reflector products of the SHF fitting loop,
 *   eq:ak / eq:bk: A_k = (U_{k-1}...U_1) DSD (U_1...U_{k-1}) is HH_OP_T
 *   with U = [u_1 .. u_{k-1}] and M = DSD.  Computed as two hh_apply passes around a
 *   batched transpose ((op(Q) (op(Q) M)^T)^T); M need not be symmetric.
 *   workspace (DEVICE) >= hh_workspace_bytes(HH_CALL_CONGRUENCE, n, h, count, 0, dtype)
 *   (two n*n*count scratch matrices + the apply's own scratch).  M_out may alias M.
 */
hh_status hh_congruence(hh_op op, int64_t n, int64_t h, const void *U, const void *M, void *Mout,
                        int64_t count, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                        hh_stream_t stream);

/*
 * hh_shf_cost -- the SHF fitting objective of one reflector and its gradient for K
 *   candidate vectors u_k (NEXT-f4):
 *     cost[k]   = C(u_k) = u^T (A B + B A) u - 2 tr(A u u^T B u u^T)       (eq:theRk)
 *               = 2 (A u)^T (B u) - 2 (u^T A u)(u^T B u)                    (A, B symmetric)
 *     grad[:,k] = 2 (A B + B A) u - 4 ((u^T A u) B + (u^T B u) A) u        (eq:gradient)
 *   the per-candidate quantities of the SHF step: the gamma sweep of eq:combine and the
 *   gradient iteration eq:iterate evaluate C (and grad C) at many u for one (A_k, B_k).
 *   A, B: n x n SYMMETRIC (DEVICE; symmetry is a documented, unvalidated precondition --
 *   either storage order then reads the same), Uc: n x K column-major (u_k at Uc + k n),
 *   cost: K values, grad: n x K column-major or NULL (cost only).  u need not be unit.
 *   Computed as [A u | B u] for all k (one batched contraction), per-candidate dots, and
 *   (with grad) A (B u) + B (A u) with the -4 (.) terms fused; A B + B A is never formed.
 *   fp32 or fp64 on the FMA pipe.  workspace (DEVICE) >=
 *   hh_workspace_bytes(HH_CALL_SHF, n, 0, K, 0, dtype) (a = A u and b = B u for every
 *   candidate, the split-K partial products of the contraction, a few per-candidate scalars).  Errors: HH_ERR_INVALID_VALUE (n < 1, K < 0, NULL operands, bad dtype),
 *   HH_ERR_WORKSPACE (too small), HH_ERR_UNSUPPORTED (operands not aligned to the dtype).
 */
hh_status hh_shf_cost(int64_t n, const void *A, const void *B, const void *Uc, int64_t K,
                      void *cost, void *grad, hh_dtype dtype, void *workspace,
                      size_t workspace_bytes, hh_stream_t stream);

/*
 * hh_knn -- test-time k nearest neighbours under the learned metric (NEXT-f3):
 *   "perform the transformation x <- L x before running the k-NN",
 *   L = diag(sqrt d) Q^T (reading R4), so d_S(q, r) = ||L x_q - L x_r||^2.
 *   For every query q (column of P_query, n x M_query column-major) return the k
 *   references (columns of P_ref, n x M_ref) with the smallest d_S, ascending, ties by
 *   the smaller reference index: nn_idx[q*k + t] (int32), nn_dist[q*k + t] (dtype).
 *   Each point is transformed once (fused kernel), then distances
 *   ||z_q||^2 + ||z_r||^2 - 2 z_q.z_r run on the tcgen05 tensor cores (bf16x3 split,
 *   fp32 accumulation) with a fused per-query top-k.
 *   v1 limits (HH_ERR_UNSUPPORTED otherwise): fp32, n <= 256, 1 <= k <= 16 (any such n:
 *   the transform of points whose rows are not 16-byte strided runs on K1g).
 *   HH_ERR_INVALID_VALUE: M_ref < k, NULL operands.  workspace (DEVICE) >=
 *   hh_workspace_bytes(HH_CALL_KNN, n, h, M_ref, M_query, dtype).
 */
hh_status hh_knn(int64_t n, int64_t h, const void *U, const void *d, const void *P_ref,
                 int64_t M_ref, const void *P_query, int64_t M_query, int k, int32_t *nn_idx,
                 void *nn_dist, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                 hh_stream_t stream);

/*
 * hh_apply_host -- hh_apply with HOST U, X, Y (end-to-end path).
 *   Streams column chunks host -> device, applies Q or Q^T with the same fused
 *   kernel, and streams them back, overlapping H2D copy, compute and D2H copy on
 *   internal streams ordered after `stream`.  Synchronous: returns after Y is
 *   written.  Host buffers should be page-locked for full PCIe bandwidth.
 *   workspace: DEVICE scratch >= hh_workspace_bytes(HH_CALL_APPLY_HOST, n, h, N, 0,
 *   dtype) (U plus a ring of column chunks; the ring is <= 3 x 64 MiB).
 */
hh_status hh_apply_host(hh_op op, int64_t n, int64_t h, const void *U_host,
                        const void *X_host, void *Y_host, int64_t N, hh_dtype dtype,
                        void *workspace, size_t workspace_bytes, hh_stream_t stream);

/*
 * hh_set_algo -- select the hh_apply path for subsequent calls of the calling
 * thread (thread-local; default HH_ALGO_AUTO).  HH_ERR_INVALID_VALUE for an
 * unknown value.  hh_get_algo returns the current selection.
 */
hh_status hh_set_algo(hh_algo algo);
hh_algo hh_get_algo(void);
/* (hh_set_algo applies to hh_apply and hh_sym_apply.) */

/*
 * hh_workspace_bytes -- scratch bytes the call needs (cuBLAS bufferSize style).
 *   N_or_M: N for apply/sym/apply_host, M for Mahalanobis, M_ref for kNN (with
 *   npairs = M_query), the matrix count for the congruence.  Writes *bytes.
 *   HH_CALL_APPLY: the compact-WY scratch when this thread's hh_algo selection
 *   picks K5 for (n, h, N, dtype) (packed W, T, V = W T and one G block), else 0.
 *   HH_CALL_SYM: the compact-WY scratch when the symmetric call picks the tensor-core
 *   block program, else 0.  HH_CALL_MAHALANOBIS: n*M*sizeof(dtype) (the
 *   transform-once Z) + the pair buckets (2 M + (M+1) + npairs + ceil(M/4096) int32,
 *   each 256-B rounded).  Errors: HH_ERR_INVALID_VALUE for bad arguments.
 */
hh_status hh_workspace_bytes(hh_call call, int64_t n, int64_t h, int64_t N_or_M,
                             int64_t npairs, hh_dtype dtype, size_t *bytes);

/* Static string for a status code (never NULL). */
const char *hh_status_string(hh_status s);

/* Library version as "MAJOR.MINOR.PATCH" (static string). */
const char *hh_version(void);

/*
 * hh_last_launch_info -- diagnostics of the calling thread's last launch of the
 * fused kernel: the kernel variant name (static string), grid, block, dynamic
 * shared-memory bytes and number of reflector chunks.  Any out pointer may be
 * NULL.  Returns HH_ERR_INVALID_VALUE if this thread launched nothing yet.
 */
hh_status hh_last_launch_info(const char **variant, int *grid, int *block,
                              int *smem_bytes, int *nchunks);

/* Number of kernels the calling thread's last call enqueued (all of them this
 * library's own).  HH_ERR_INVALID_VALUE before any launch or for a NULL pointer. */
hh_status hh_last_launch_count(int *kernels);

#ifdef __cplusplus
}
#endif

#endif /* HH_H_ */
