// hh_cong.cu -- NEXT-f4: the two-sided reflector application (congruence) that the
// SHF fitting loop is built from:
//
//   A_k = (U_{k-1} ... U_1) D S D (U_1 ... U_{k-1})   = Q^T M Q,  Q = H_1 ... H_{k-1}
//   B_k = (U_{k+1} ... U_h) diag(s) (U_h ... U_{k+1}) = Q' diag(s) Q'^T
//
// hh_congruence computes M_out = op(Q) M op(Q)^T for a batch of n x n column-major
// matrices as  Y = op(Q) M  (apply to the n*count columns), a batched transpose,
// op(Q) again, and a transpose back:  (op(Q) (op(Q) M)^T)^T = op(Q) M op(Q)^T.
// The applies are the library's K1 / K5 kernels; the transpose is a 32 x 32
// shared-memory tiled kernel (one read and one write of each matrix).
#include <cuda_runtime.h>

#include <algorithm>

#include "hh_internal.h"

namespace hh {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) batched_transpose_kernel(const T *__restrict__ A,
                                                                T *__restrict__ B, int64_t n) {
    __shared__ T tile[32][33];
    const int64_t base = static_cast<int64_t>(blockIdx.z) * n * n;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    // A is column-major: element (r, c) at c*n + r
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, r = r0 + tx;
        if (c < n && r < n) tile[k][tx] = A[base + c * n + r];
    }
    __syncthreads();
    // B(c, r) = A(r, c): B column r holds A's row r
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k, c = c0 + tx;
        if (c < n && r < n) B[base + r * n + c] = tile[tx][k];
    }
}

}  // namespace

cudaError_t launch_transpose(const void *A, void *B, int64_t n, int64_t count, int dtype,
                             cudaStream_t stream) {
    const unsigned g = static_cast<unsigned>((n + 31) / 32);
    const dim3 grid(g, g, static_cast<unsigned>(count));
    if (dtype == 0)
        batched_transpose_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float *>(A),
                                                                 static_cast<float *>(B), n);
    else
        batched_transpose_kernel<double><<<grid, 256, 0, stream>>>(static_cast<const double *>(A),
                                                                  static_cast<double *>(B), n);
    return cudaGetLastError();
}

}  // namespace hh
