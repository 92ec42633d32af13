/*
 * hh_ref.c -- the fp64 CPU ORACLE for the Householder-product apply path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1811_07624_b200/) never links, imports or executes it, and shares no
 * code, header, table or helper with it.
 *
 * Plain, slow, obviously correct: one column (or one pair) at a time, reflectors
 * applied one by one in the paper's order, sequential ascending-index dot
 * products, strict IEEE fp64 (build: gcc -O2 -fopenmp -ffp-contract=off, no
 * -ffast-math).  OpenMP only splits independent columns / pairs.
 *
 * Citations: P:L = /root/reference/PAPER.md line L (as pinned in SURVEY.md §0).
 *   Eq. 1  eq:thefactorization   P:42-45   Ubar = D U_h ... U_1
 *   Eq. 2  eq:theReflector       P:47-50   U_k = I - 2 u_k u_k^T, ||u_k|| = 1
 *   text                         P:54      "takes 4nh operations" (dot + update)
 *   text                         P:233-237 reflectors are symmetric (J_k^T = J_k)
 *   eq:thesbar                   P:277-284 S = Q diag(s) Q^T, "(8h+1)n operations"
 *   LMNN transform               P:600, P:668  d_S(x_i,x_j) = ||L(x_i - x_j)||^2,
 *                                              L = sqrt(Lambda) U
 *
 * Conventions (readings R1, R3, R4, R5):
 *   Q := H_1 H_2 ... H_h, H_i = I - 2 u_i u_i^T, u_i = U[i*n .. i*n+n-1]
 *   (U is n x h column-major == (h, n) row-major).  The stored u_i is used
 *   literally: no renormalisation, no tau = 2/||u||^2.
 *   op 0 (N): Y = Q X    -> apply u_h first, u_1 last   (i = h-1 ... 0)
 *   op 1 (T): Y = Q^T X  -> apply u_1 first, u_h last   (i = 0 ... h-1)
 *   X, Y: n x N column-major (column j at X + j*n).
 *
 * Parity pins: tests/test_oracle_pins.py (dense brute force, H^2 = I, norm
 * preservation, det, QR reproduction, rotation worked example, Hadamard / FWHT,
 * closed form I - 2 W W^T, eigvalsh spectrum, Mahalanobis invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* One reflector on one vector, literally x <- (I - 2 u u^T) x  (Eq. 2):
 * a = u^T x (ascending r), then x[r] -= 2 a u[r].  2n multiply-adds ("4nh"). */
static void reflect(int64_t n, const double *u, double *x) {
    double a = 0.0;
    for (int64_t r = 0; r < n; ++r) a += u[r] * x[r];
    a = 2.0 * a;
    for (int64_t r = 0; r < n; ++r) x[r] -= a * u[r];
}

/* x <- Q x (op 0) or Q^T x (op 1).  Q^T = H_h ... H_1 because each H_i is
 * symmetric, so the transpose only reverses the order. */
static void apply_one(int op, int64_t n, int64_t h, const double *U, double *x) {
    if (op == 0) {
        for (int64_t i = h - 1; i >= 0; --i) reflect(n, U + i * n, x);
    } else {
        for (int64_t i = 0; i < h; ++i) reflect(n, U + i * n, x);
    }
}

int hh_ref_apply(int op, int64_t n, int64_t h, const double *U, const double *X,
                 double *Y, int64_t N) {
    if ((op != 0 && op != 1) || n < 1 || h < 0 || N < 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)n);
        if (!x) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t j = 0; j < N; ++j) {
                memcpy(x, X + j * n, sizeof(double) * (size_t)n);
                apply_one(op, n, h, U, x);
                memcpy(Y + j * n, x, sizeof(double) * (size_t)n);
            }
            free(x);
        }
    }
    return bad ? 2 : 0;
}

/* Y = Q diag(lambda) Q^T X  (eq:thesbar, with D = I, reading R2):
 * first the Q^T pass (u_1 first), then x[r] *= lambda[r], then the Q pass
 * (u_h first): two reflector passes plus one diagonal scale, (8h+1)n ops. */
int hh_ref_sym_apply(int64_t n, int64_t h, const double *U, const double *lam,
                     const double *X, double *Y, int64_t N) {
    if (n < 1 || h < 0 || N < 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)n);
        if (!x) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t j = 0; j < N; ++j) {
                memcpy(x, X + j * n, sizeof(double) * (size_t)n);
                apply_one(1, n, h, U, x);
                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];
                apply_one(0, n, h, U, x);
                memcpy(Y + j * n, x, sizeof(double) * (size_t)n);
            }
            free(x);
        }
    }
    return bad ? 2 : 0;
}

/* dist[j] = || D^{1/2} Q^T (P[:,ia[j]] - P[:,ib[j]]) ||^2
 *         = sum_r d[r] * (Q^T z)_r^2,   z = x_a - x_b
 * (P:600 d_S = ||L(x_i - x_j)||^2; P:668 L = sqrt(Lambda) U with U == Q^T,
 * reading R4).  The literal per-pair form: the difference is formed first,
 * then transformed -- the GPU's transform-once rearrangement is NOT copied. */
int hh_ref_mahalanobis(int64_t n, int64_t h, const double *U, const double *d,
                       const double *P, int64_t M, const int32_t *ia,
                       const int32_t *ib, int64_t npairs, double *dist) {
    if (n < 1 || h < 0 || npairs < 0 || (npairs > 0 && M < 1)) return 1;
    for (int64_t j = 0; j < npairs; ++j)
        if (ia[j] < 0 || ia[j] >= M || ib[j] < 0 || ib[j] >= M) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *z = (double *)malloc(sizeof(double) * (size_t)n);
        if (!z) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t j = 0; j < npairs; ++j) {
                const double *xa = P + (int64_t)ia[j] * n;
                const double *xb = P + (int64_t)ib[j] * n;
                for (int64_t r = 0; r < n; ++r) z[r] = xa[r] - xb[r];
                apply_one(1, n, h, U, z);
                double s = 0.0;
                for (int64_t r = 0; r < n; ++r) s += d[r] * (z[r] * z[r]);
                dist[j] = s;
            }
            free(z);
        }
    }
    return bad ? 2 : 0;
}

/* NEXT-f1: the paper's exact forms with the diagonal D = diag(d) of Eq. 1.
 * side 0 (left, Eq. 1 / eq:thesbar):   Y = D op(Q) X
 * side 1 (right, Result 3):  Y = op(Q) D X
 * Written out literally: scale, then the same reflector-by-reflector apply. */
int hh_ref_apply_signed(int op, int side, int64_t n, int64_t h, const double *U,
                        const double *d, const double *X, double *Y, int64_t N) {
    if ((op != 0 && op != 1) || (side != 0 && side != 1) || n < 1 || h < 0 || N < 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)n);
        if (!x) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t j = 0; j < N; ++j) {
                memcpy(x, X + j * n, sizeof(double) * (size_t)n);
                if (side == 1)
                    for (int64_t r = 0; r < n; ++r) x[r] *= d[r];
                apply_one(op, n, h, U, x);
                if (side == 0)
                    for (int64_t r = 0; r < n; ++r) x[r] *= d[r];
                memcpy(Y + j * n, x, sizeof(double) * (size_t)n);
            }
            free(x);
        }
    }
    return bad ? 2 : 0;
}

/* S-bar X = D Q diag(lambda) Q^T D X  (eq:thesbar, D on both sides). */
int hh_ref_sym_apply_signed(int64_t n, int64_t h, const double *U, const double *d,
                            const double *lam, const double *X, double *Y, int64_t N) {
    if (n < 1 || h < 0 || N < 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)n);
        if (!x) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t j = 0; j < N; ++j) {
                memcpy(x, X + j * n, sizeof(double) * (size_t)n);
                for (int64_t r = 0; r < n; ++r) x[r] *= d[r];
                apply_one(1, n, h, U, x);
                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];
                apply_one(0, n, h, U, x);
                for (int64_t r = 0; r < n; ++r) x[r] *= d[r];
                memcpy(Y + j * n, x, sizeof(double) * (size_t)n);
            }
            free(x);
        }
    }
    return bad ? 2 : 0;
}

/* NEXT-f3: k nearest references of each query under d_S:
 * d_S(q, r) = || D^{1/2} Q^T (x_q - x_r) ||^2, the literal per-pair form of
 * hh_ref_mahalanobis for every (query, reference) pair, then the k smallest in
 * ascending (distance, reference index) order. */
int hh_ref_knn(int64_t n, int64_t h, const double *U, const double *d, const double *Pr,
               int64_t Mr, const double *Pq, int64_t Mq, int k, int32_t *idx, double *dist) {
    if (n < 1 || h < 0 || Mr < k || Mq < 0 || k < 1) return 1;
    int bad = 0;
#pragma omp parallel
    {
        double *z = (double *)malloc(sizeof(double) * (size_t)n);
        double *bd = (double *)malloc(sizeof(double) * (size_t)k);
        int32_t *bi = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
        if (!z || !bd || !bi) {
#pragma omp atomic write
            bad = 1;
        } else {
#pragma omp for schedule(dynamic, 4)
            for (int64_t q = 0; q < Mq; ++q) {
                int cnt = 0;
                for (int64_t r = 0; r < Mr; ++r) {
                    for (int64_t e = 0; e < n; ++e) z[e] = Pq[q * n + e] - Pr[r * n + e];
                    apply_one(1, n, h, U, z);
                    double s = 0.0;
                    for (int64_t e = 0; e < n; ++e) s += d[e] * (z[e] * z[e]);
                    if (cnt == k && !(s < bd[k - 1])) continue;   /* ties keep the earlier r */
                    int pos = cnt < k ? cnt : k - 1;
                    while (pos > 0 && bd[pos - 1] > s) {
                        bd[pos] = bd[pos - 1];
                        bi[pos] = bi[pos - 1];
                        --pos;
                    }
                    bd[pos] = s;
                    bi[pos] = (int32_t)r;
                    if (cnt < k) ++cnt;
                }
                for (int t = 0; t < k; ++t) {
                    idx[q * k + t] = bi[t];
                    dist[q * k + t] = bd[t];
                }
            }
        }
        free(z);
        free(bd);
        free(bi);
    }
    return bad ? 2 : 0;
}

/* NEXT-f4: M_out = op(Q) M op(Q)^T for `count` n x n column-major matrices (the
 * congruences A_k, B_k of eq:ak / eq:bk), literally: apply op(Q) to every
 * column of M, transpose, apply again, transpose back. */
int hh_ref_congruence(int op, int64_t n, int64_t h, const double *U, const double *M,
                      double *Mout, int64_t count) {
    if ((op != 0 && op != 1) || n < 1 || h < 0 || count < 0) return 1;
    const size_t nn = (size_t)n * (size_t)n;
    double *A = (double *)malloc(sizeof(double) * nn);
    double *B = (double *)malloc(sizeof(double) * nn);
    if (!A || !B) {
        free(A);
        free(B);
        return 2;
    }
    int rc = 0;
    for (int64_t b = 0; b < count && !rc; ++b) {
        rc = hh_ref_apply(op, n, h, U, M + (size_t)b * nn, A, n);     /* A = op(Q) M */
        for (int64_t c = 0; c < n; ++c)                              /* B = A^T */
            for (int64_t r = 0; r < n; ++r) B[c * n + r] = A[r * n + c];
        if (!rc) rc = hh_ref_apply(op, n, h, U, B, A, n);             /* A = op(Q) B */
        for (int64_t c = 0; c < n; ++c)                              /* out = A^T */
            for (int64_t r = 0; r < n; ++r) Mout[(size_t)b * nn + c * n + r] = A[r * n + c];
    }
    free(A);
    free(B);
    return rc;
}

/* NEXT-f4: the SHF objective of one reflector and its gradient for K
 * candidate vectors u_k (Uc: n x K column-major, u_k = Uc + k*n), A and B symmetric n x n:
 *   C(u)      = u^T (A B + B A) u - 2 tr(A u u^T B u u^T)                   eq:theRk
 *   tr(A u u^T B u u^T) = (u^T A u)(u^T B u)                               (cyclic trace)
 *   grad C(u) = 2 (A B + B A) u - 4 ((u^T A u) B + (u^T B u) A) u           eq:gradient
 * Literally: the matrix A B + B A is formed once (plain triple loop), then each candidate
 * takes its quadratic forms and matrix-vector products one by one.  grad may be NULL. */
int hh_ref_shf_cost(int64_t n, const double *A, const double *B, const double *Uc, int64_t K,
                    double *cost, double *grad) {
    if (n < 1 || K < 0) return 1;
    const size_t nn = (size_t)n * (size_t)n;
    double *Mab = (double *)malloc(sizeof(double) * nn);
    if (!Mab) return 2;
    /* Mab = A B + B A (entry (i, j); A, B symmetric so either storage order) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t l = 0; l < n; ++l) s += A[i * n + l] * B[l * n + j];
            for (int64_t l = 0; l < n; ++l) s += B[i * n + l] * A[l * n + j];
            Mab[i * n + j] = s;
        }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < K; ++k) {
        const double *u = Uc + (size_t)k * (size_t)n;
        double q = 0.0, qa = 0.0, qb = 0.0;   /* u^T Mab u, u^T A u, u^T B u */
        for (int64_t i = 0; i < n; ++i) {
            double mi = 0.0, ai = 0.0, bi = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                mi += Mab[i * n + j] * u[j];
                ai += A[i * n + j] * u[j];
                bi += B[i * n + j] * u[j];
            }
            q += u[i] * mi;
            qa += u[i] * ai;
            qb += u[i] * bi;
        }
        cost[k] = q - 2.0 * (qa * qb);
        if (grad) {
            double *g = grad + (size_t)k * (size_t)n;
            for (int64_t i = 0; i < n; ++i) {
                double mi = 0.0, ci = 0.0;
                for (int64_t j = 0; j < n; ++j) {
                    mi += Mab[i * n + j] * u[j];
                    ci += (qa * B[i * n + j] + qb * A[i * n + j]) * u[j];
                }
                g[i] = 2.0 * mi - 4.0 * ci;
            }
        }
    }
    free(Mab);
    return 0;
}

int hh_ref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void hh_ref_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
