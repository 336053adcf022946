// Setup (outside the timed region): factorisations and the composite
// operators the hot-path kernels apply.  cuSOLVER getrf/getrs + cuBLAS are used here
// only; the per-step work runs in libpe's own kernels.
//
//   sequential (stepping.py:109-147): with K = M11/dt + A11,
//     u+ = Pu u + Pa w + Pd (w - w_prev) + cu
//     w+ = Ew w + Qd (u - u_prev) + Qu u+ + cw
//   where Pu = K^-1 M11/dt, Pa = -K^-1 A12, Pd = -K^-1 M12/dt, cu = K^-1 f1,
//         Ew = I - dt M22^-1 A22, Qd = -M22^-1 M12^T, Qu = -dt M22^-1 A12^T, cw = dt M22^-1 f2.
//   Substituting u+ gives one (d x 2d) operator T acting on [u; w; u-u_prev; w-w_prev]:
//     T = [[Pu,     Pa,         0,  Pd    ],
//          [Qu Pu,  Ew + Qu Pa, Qd, Qu Pd ]],   c = [cu; cw + Qu cu].
//   coarse (stepping.py:149-176): G(x) = Phi x + gG with Phi = K_G^-1 R_G, gG = K_G^-1 f.
//   all-at-once (allatonce.py:100-110, 184-210): shifted inverses (d_k M11 + A11)^-1 as
//     real 2x2-block matrices, the rhs operator [-A12 | -M12/dt] on [w_s; w_s - w_{s-1}]
//     (difference first, as build_rhs does), M11/dt,
//     the w-sweep operator [-dt M22^-T A12^T | -M22^-T M12^T], dt M22^-T f2, E and the
//     alpha-circulant time transforms S^-1 (2J x J) and Re(S .) (J x 2J).

#include <cuComplex.h>

#include <cmath>
#include <complex>
#include <vector>

#include "pe.h"
#include "pe_ctx.h"

namespace pe {

#define BLAS_CHECK(x)                                                               \
  do {                                                                              \
    cublasStatus_t _s = (x);                                                        \
    if (_s != CUBLAS_STATUS_SUCCESS)                                                \
      throw Error{PE_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(_s)}; \
  } while (0)
#define SOLVER_CHECK(x)                                                             \
  do {                                                                              \
    cusolverStatus_t _s = (x);                                                      \
    if (_s != CUSOLVER_STATUS_SUCCESS)                                              \
      throw Error{PE_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(_s)}; \
  } while (0)

// row-major C(m x n) = alpha op(A) op(B) + beta C
static void rm_gemm(cublasHandle_t h, bool tA, bool tB, int m, int n, int k, double alpha,
                    const double* A, int lda, const double* B, int ldb, double beta, double* C,
                    int ldc) {
  if (m == 0 || n == 0) return;
  if (k == 0) {
    // C = beta C: scale via geam
    BLAS_CHECK(cublasDgeam(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, &beta, C, ldc, &beta, C, ldc, C,
                           ldc));
    double zero = 0.0;
    if (beta == 0.0)
      BLAS_CHECK(cublasDgeam(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, &zero, C, ldc, &zero, C, ldc, C,
                             ldc));
    return;
  }
  BLAS_CHECK(cublasDgemm(h, tB ? CUBLAS_OP_T : CUBLAS_OP_N, tA ? CUBLAS_OP_T : CUBLAS_OP_N, n,
                         m, k, &alpha, B, ldb, A, lda, &beta, C, ldc));
}
// row-major C(m x n) = alpha op(A) + beta op(B)
static void rm_geam(cublasHandle_t h, bool tA, bool tB, int m, int n, double alpha,
                    const double* A, int lda, double beta, const double* B, int ldb, double* C,
                    int ldc) {
  if (m == 0 || n == 0) return;
  BLAS_CHECK(cublasDgeam(h, tA ? CUBLAS_OP_T : CUBLAS_OP_N, tB ? CUBLAS_OP_T : CUBLAS_OP_N, n,
                         m, &alpha, A, lda, &beta, B, ldb, C, ldc));
}

__global__ void set_identity_kernel(int n, double* X, int ld, double scale) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = (long long)n * n;
  for (; t < tot; t += (long long)gridDim.x * blockDim.x) {
    int i = (int)(t / n), j = (int)(t % n);
    X[(long long)i * ld + j] = (i == j) ? scale : 0.0;
  }
}
static void set_identity(int n, double* X, int ld, double scale, cudaStream_t st) {
  if (n == 0) return;
  set_identity_kernel<<<std::min(1024, (n * n + 255) / 256), 256, 0, st>>>(n, X, ld, scale);
  PE_CUDA_CHECK(cudaGetLastError());
}

__global__ void zero_block_kernel(int m, int n, double* X, int ld) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; t < (long long)m * n; t += (long long)gridDim.x * blockDim.x)
    X[(t / n) * ld + (t % n)] = 0.0;
}

// The shifted matrix d_k M11 + A11 in its real block form [[Re, -Im], [Im, Re]] (2n x 2n
// row-major): its inverse is the block form of the complex inverse, i.e. the operator the
// sweep applies to the planar (re, im) transformed right-hand sides.
__global__ void shifted_blockform_kernel(int n, double dre, double dim, const double* M,
                                         const double* A, double* S) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n2 = 2LL * n;
  for (; t < (long long)n * n; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t % n;
    const double re = dre * M[t] + A[t], im = dim * M[t];
    S[i * n2 + j] = re;
    S[i * n2 + n + j] = -im;
    S[(i + n) * n2 + j] = im;
    S[(i + n) * n2 + n + j] = re;
  }
}
// The real modes k = 0 and (J even) k = J/2 share pseudo-mode 0 as a block diagonal;
// a missing second mode (J odd) is an identity block, cleared again after the inversion.
__global__ void shifted_real_block_kernel(int n, double dre, const double* M, const double* A,
                                          double* S, int which, int identity) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n2 = 2LL * n, o = (long long)which * n;
  for (; t < (long long)n * n; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t % n;
    S[(i + o) * n2 + o + j] = identity ? (i == j ? 1.0 : 0.0) : dre * M[t] + A[t];
  }
}
__global__ void clear_block_kernel(int n, double* S, int which) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n2 = 2LL * n, o = (long long)which * n;
  for (; t < (long long)n * n; t += (long long)gridDim.x * blockDim.x)
    S[(t / n + o) * n2 + o + t % n] = 0.0;
}

__global__ void transpose_blocks_kernel(int nblocks, int n, const double* src, double* dst) {
  const long long per = (long long)n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < per * nblocks;
       t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / per, r = t - b * per;
    const long long i = r / n, j = r - i * n;
    dst[b * per + j * n + i] = src[t];
  }
}

void transpose_blocks(int nblocks, int n, const double* src, double* dst, cudaStream_t st) {
  const long long tot = (long long)n * n * nblocks;
  if (tot == 0) return;
  transpose_blocks_kernel<<<(int)std::min<long long>(4096, (tot + 255) / 256), 256, 0, st>>>(
      nblocks, n, src, dst);
  PE_CUDA_CHECK(cudaGetLastError());
}

static int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>(4096, (n + 255) / 256)); }

// Ainv = A^{-1} for a row-major n x n buffer: libpe's own blocked LU (batchlu.cu).
static void inverse(pe_ctx* c, int n, const double* A, double* Ainv) {
  if (n == 0) return;
  cudaStream_t st = c->setup_stream;
  DevBuf lu, ipiv, info;
  lu.ensure(sizeof(double) * n * (size_t)n);
  ipiv.ensure(sizeof(int) * n);
  info.ensure(sizeof(int));
  PE_CUDA_CHECK(cudaMemcpyAsync(lu.p, A, sizeof(double) * n * (size_t)n, cudaMemcpyDeviceToDevice, st));
  batched_lu_inverse(n, 1, lu.d(), Ainv, ipiv.i(), info.i(), st);
  int h_info = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h_info != 0) throw Error{PE_ERR_SOLVER, "singular matrix in setup factorisation (zero pivot " + std::to_string(h_info) + ")"};
}

void setup_sequential(pe_ctx* c, double dt) {
  const int d1 = c->d1, d2 = c->d2, d = c->d;
  cudaStream_t st = c->setup_stream;
  cublasHandle_t h = c->blas;
  c->T.ensure(sizeof(double) * (size_t)c->E * d * 2 * d + 8);
  c->cvec.ensure(sizeof(double) * (size_t)c->E * d + 8);
  c->Lf.ensure(sizeof(double) * (size_t)c->E * d * d + 8);
  DevBuf K, Kinv, M22inv, Ew, Qd, Qu, cw;
  K.ensure(sizeof(double) * d1 * (size_t)d1 + 8);
  Kinv.ensure(sizeof(double) * d1 * (size_t)d1 + 8);
  M22inv.ensure(sizeof(double) * d2 * (size_t)d2 + 8);
  Ew.ensure(sizeof(double) * d2 * (size_t)d2 + 8);
  Qd.ensure(sizeof(double) * d2 * (size_t)d1 + 8);
  Qu.ensure(sizeof(double) * d2 * (size_t)d1 + 8);
  cw.ensure(sizeof(double) * d2 + 8);
  const int ldT = 2 * d;
  for (int e = 0; e < c->E; ++e) {
    const double* M11 = c->M11.d() + (size_t)e * d1 * d1;
    const double* A11 = c->A11.d() + (size_t)e * d1 * d1;
    const double* M12 = c->M12.d() + (size_t)e * d1 * d2;
    const double* A12 = c->A12.d() + (size_t)e * d1 * d2;
    const double* M22 = c->M22.d() + (size_t)e * d2 * d2;
    const double* A22 = c->A22.d() + (size_t)e * d2 * d2;
    const double* f1 = c->f1.d() + (size_t)e * d1;
    const double* f2 = c->f2.d() + (size_t)e * d2;
    double* T = c->T.d() + (size_t)e * d * ldT;
    double* cv = c->cvec.d() + (size_t)e * d;
    // load map: bias = Lf [f1; f2], Lf = [[K^-1, 0], [Qu K^-1, dt M22^-1]] (the loads'
    // path through split_step, stepping.py:125-146), for time-dependent loads
    double* Lf = c->Lf.d() + (size_t)e * d * d;
    zero_block_kernel<<<grid_for((long long)d * d), 256, 0, st>>>(d, d, Lf, d);
    zero_block_kernel<<<grid_for((long long)d * ldT), 256, 0, st>>>(d, ldT, T, ldT);
    if (d1) {
      rm_geam(h, false, false, d1, d1, 1.0 / dt, M11, d1, 1.0, A11, d1, K.d(), d1);
      inverse(c, d1, K.d(), Kinv.d());
      rm_gemm(h, false, false, d1, d1, d1, 1.0 / dt, Kinv.d(), d1, M11, d1, 0.0, T, ldT);  // Pu
      if (d2) {
        rm_gemm(h, false, false, d1, d2, d1, -1.0, Kinv.d(), d1, A12, d2, 0.0, T + d1, ldT);  // Pa
        rm_gemm(h, false, false, d1, d2, d1, -1.0 / dt, Kinv.d(), d1, M12, d2, 0.0,
                T + d + d1, ldT);  // Pd
      }
      rm_gemm(h, false, false, d1, 1, d1, 1.0, Kinv.d(), d1, f1, 1, 0.0, cv, 1);  // cu
      rm_geam(h, false, false, d1, d1, 1.0, Kinv.d(), d1, 0.0, Kinv.d(), d1, Lf, d);
    }
    if (d2) {
      inverse(c, d2, M22, M22inv.d());
      double* Tw = T + (size_t)d1 * ldT;  // rows d1..d-1
      // Ew = I - dt M22^-1 A22 written straight into T[d1:, d1:d]
      set_identity(d2, Tw + d1, ldT, 1.0, st);
      rm_gemm(h, false, false, d2, d2, d2, -dt, M22inv.d(), d2, A22, d2, 1.0, Tw + d1, ldT);
      rm_gemm(h, false, false, d2, 1, d2, dt, M22inv.d(), d2, f2, 1, 0.0, cv + d1, 1);  // cw
      rm_geam(h, false, false, d2, d2, dt, M22inv.d(), d2, 0.0, M22inv.d(), d2,
              Lf + (size_t)d1 * d + d1, d);
      if (d1) {
        rm_gemm(h, false, true, d2, d1, d2, -1.0, M22inv.d(), d2, M12, d2, 0.0, Tw + d, ldT);  // Qd
        rm_gemm(h, false, true, d2, d1, d2, -dt, M22inv.d(), d2, A12, d2, 0.0, Qu.d(), d1);   // Qu
        // fold u+ into the w rows: Qu [Pu, Pa, 0, Pd] and Qu cu
        rm_gemm(h, false, false, d2, d1, d1, 1.0, Qu.d(), d1, T, ldT, 0.0, Tw, ldT);
        rm_gemm(h, false, false, d2, d2, d1, 1.0, Qu.d(), d1, T + d1, ldT, 1.0, Tw + d1, ldT);
        rm_gemm(h, false, false, d2, d2, d1, 1.0, Qu.d(), d1, T + d + d1, ldT, 0.0,
                Tw + d + d1, ldT);
        rm_gemm(h, false, false, d2, 1, d1, 1.0, Qu.d(), d1, cv, 1, 1.0, cv + d1, 1);
        rm_gemm(h, false, false, d2, d1, d1, 1.0, Qu.d(), d1, Kinv.d(), d1, 0.0,
                Lf + (size_t)d1 * d, d);
      }
    }
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  c->seq_dt = dt;
}

__global__ void assemble_coarse_kernel(int d1, int d2, double dt, const double* M11,
                                       const double* A11, const double* M12, const double* A12,
                                       const double* M22, const double* A22, double* KG,
                                       double* RG) {
  const int d = d1 + d2;
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; t < (long long)d * d; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / d), j = (int)(t % d);
    double k, r;
    if (i < d1 && j < d1) {
      const double m = M11[i * d1 + j], a = A11[i * d1 + j];
      k = m / dt + a;
      r = m / dt;
    } else if (i < d1) {
      const double m = M12[i * d2 + (j - d1)], a = A12[i * d2 + (j - d1)];
      k = m / dt;
      r = m / dt - a;
    } else if (j < d1) {
      const double m = M12[j * d2 + (i - d1)], a = A12[j * d2 + (i - d1)];  // transposes
      k = m / dt + a;
      r = m / dt;
    } else {
      const double m = M22[(i - d1) * d2 + (j - d1)], a = A22[(i - d1) * d2 + (j - d1)];
      k = m / dt;
      r = m / dt - a;
    }
    KG[t] = k;
    RG[t] = r;
  }
}

void setup_coarse(pe_ctx* c, double dt) {
  const int d1 = c->d1, d2 = c->d2, d = c->d;
  cudaStream_t st = c->setup_stream;
  c->Phi.ensure(sizeof(double) * (size_t)c->E * d * d + 8);
  c->gG.ensure(sizeof(double) * (size_t)c->E * d + 8);
  c->LG.ensure(sizeof(double) * (size_t)c->E * d * d + 8);  // K_G^-1 (time-dependent loads)
  DevBuf KG, RG, KGinv, f;
  KG.ensure(sizeof(double) * (size_t)d * d);
  RG.ensure(sizeof(double) * (size_t)d * d);
  KGinv.ensure(sizeof(double) * (size_t)d * d);
  f.ensure(sizeof(double) * d);
  for (int e = 0; e < c->E; ++e) {
    assemble_coarse_kernel<<<grid_for((long long)d * d), 256, 0, st>>>(
        d1, d2, dt, c->M11.d() + (size_t)e * d1 * d1, c->A11.d() + (size_t)e * d1 * d1,
        c->M12.d() + (size_t)e * d1 * d2, c->A12.d() + (size_t)e * d1 * d2,
        c->M22.d() + (size_t)e * d2 * d2, c->A22.d() + (size_t)e * d2 * d2, KG.d(), RG.d());
    PE_CUDA_CHECK(cudaGetLastError());
    if (d1) PE_CUDA_CHECK(cudaMemcpyAsync(f.d(), c->f1.d() + (size_t)e * d1, sizeof(double) * d1, cudaMemcpyDeviceToDevice, st));
    if (d2) PE_CUDA_CHECK(cudaMemcpyAsync(f.d() + d1, c->f2.d() + (size_t)e * d2, sizeof(double) * d2, cudaMemcpyDeviceToDevice, st));
    inverse(c, d, KG.d(), KGinv.d());
    rm_gemm(c->blas, false, false, d, d, d, 1.0, KGinv.d(), d, RG.d(), d, 0.0,
            c->Phi.d() + (size_t)e * d * d, d);
    rm_gemm(c->blas, false, false, d, 1, d, 1.0, KGinv.d(), d, f.d(), 1, 0.0,
            c->gG.d() + (size_t)e * d, 1);
    PE_CUDA_CHECK(cudaMemcpyAsync(c->LG.d() + (size_t)e * d * d, KGinv.d(),
                                  sizeof(double) * (size_t)d * d, cudaMemcpyDeviceToDevice, st));
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  c->coarse_dt = dt;
}

// Modal form of the w recursion w_{s+1} = E w_s + g_s (allatonce.py:226-229).
// E = I - dt M22^-1 A22 is similar to a symmetric matrix when A22 is symmetric and M22 is
// SPD: with the M22-orthonormal eigenvectors V of the pencil A22 v = mu M22 v
// (V^T M22 V = I), E = V diag(lam) V^-1 with lam = 1 - dt mu and V^-1 = V^T M22.  In
// z = V^-1 w the J-step chain decouples into d2 scalar recurrences z_{s+1} = lam z_s + h_s,
// h_s = V^-1 g_s, so the sequential-in-time part of a sweep becomes an elementwise scan and
// W = V Z one parallel GEMM.  The decomposition is accepted only when V diag(lam) V^-1
// reproduces the E the reference forms (`e_mat`, :207) to 1e-9 relative in max norm; a
// non-symmetric A22 or indefinite M22 fails that check and keeps the direct recursion.
static bool setup_modal(pe_ctx* c, int e, double dt, const double* M22, const double* A22,
                        const double* Em, const double* GW, const double* cg) {
  const int d1 = c->d1, n = c->d2;
  cudaStream_t st = c->setup_stream;
  cublasHandle_t h = c->blas;
  DevBuf A, B, W, info, work, Vl, Er;
  A.ensure(sizeof(double) * (size_t)n * n);
  B.ensure(sizeof(double) * (size_t)n * n);
  W.ensure(sizeof(double) * n);
  info.ensure(sizeof(int));
  PE_CUDA_CHECK(cudaMemcpyAsync(A.p, A22, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, st));
  PE_CUDA_CHECK(cudaMemcpyAsync(B.p, M22, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, st));
  int lwork = 0;
  SOLVER_CHECK(cusolverDnDsygvd_bufferSize(c->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                           CUBLAS_FILL_MODE_LOWER, n, A.d(), n, B.d(), n, W.d(), &lwork));
  work.ensure(sizeof(double) * std::max(lwork, 1));
  SOLVER_CHECK(cusolverDnDsygvd(c->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                CUBLAS_FILL_MODE_LOWER, n, A.d(), n, B.d(), n, W.d(), work.d(),
                                lwork, info.i()));
  int h_info = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h_info != 0) return false;  // M22 not positive definite (or no convergence)
  // A now holds the eigenvectors column-major, i.e. V^T when read row-major
  double* V = c->Vm.d() + (size_t)e * n * n;
  double* Vi = c->Vinv.d() + (size_t)e * n * n;
  double* lam = c->lam.d() + (size_t)e * n;
  rm_geam(h, true, false, n, n, 1.0, A.d(), n, 0.0, A.d(), n, V, n);
  rm_gemm(h, false, false, n, n, n, 1.0, A.d(), n, M22, n, 0.0, Vi, n);  // V^T M22
  std::vector<double> hl(n);
  PE_CUDA_CHECK(cudaMemcpyAsync(hl.data(), W.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  for (auto& x : hl) x = 1.0 - dt * x;
  PE_CUDA_CHECK(cudaMemcpyAsync(lam, hl.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  // reconstruction check against the reference-form E
  Vl.ensure(sizeof(double) * (size_t)n * n);
  Er.ensure(sizeof(double) * (size_t)n * n);
  // row-major V scaled by columns == column-major V^T scaled by rows
  BLAS_CHECK(cublasDdgmm(h, CUBLAS_SIDE_LEFT, n, n, V, n, lam, 1, Vl.d(), n));
  rm_gemm(h, false, false, n, n, n, 1.0, Vl.d(), n, Vi, n, 0.0, Er.d(), n);
  rm_geam(h, false, false, n, n, 1.0, Er.d(), n, -1.0, Em, n, Er.d(), n);
  int idiff = 0, iref = 0;
  BLAS_CHECK(cublasIdamax(h, n * n, Er.d(), 1, &idiff));
  BLAS_CHECK(cublasIdamax(h, n * n, Em, 1, &iref));
  double vdiff = 0, vref = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&vdiff, Er.d() + idiff - 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaMemcpyAsync(&vref, Em + iref - 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  if (!(std::fabs(vdiff) <= 1e-9 * std::fabs(vref))) return false;
  if (d1) rm_gemm(h, false, false, n, 2 * d1, n, 1.0, Vi, n, GW, 2 * d1, 0.0,
                  c->GZ.d() + (size_t)e * n * 2 * d1, 2 * d1);
  rm_gemm(h, false, false, n, 1, n, 1.0, Vi, n, cg, 1, 0.0, c->cgz.d() + (size_t)e * n, 1);
  return true;
}

__global__ void sub_diag_kernel(int n, double* P, int ld, const double* d, double scale) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    P[(long long)t * ld + t] -= d ? d[t] : scale;
}

static double max_abs(pe_ctx* c, long long n, const double* x) {
  if (n == 0) return 0.0;
  int idx = 0;
  BLAS_CHECK(cublasIdamax(c->blas, (int)n, x, 1, &idx));
  double v = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&v, x + idx - 1, sizeof(double), cudaMemcpyDeviceToHost, c->setup_stream));
  PE_CUDA_CHECK(cudaStreamSynchronize(c->setup_stream));
  return std::fabs(v);
}

// Generalized symmetric-definite eigenproblem A v = mu M v (cuSOLVER sygvd): V (row-major,
// eigenvectors as columns), Vi = V^T M = V^-1 and mu (host).  Accepted only if
// V^T A V = diag(mu) and V^T M V = I hold to 1e-9 (relative to max |mu| for the former):
// a non-symmetric A or an indefinite M fails here.
static bool pencil_eig(pe_ctx* c, int n, const double* A, const double* M, double* V, double* Vi,
                       std::vector<double>& mu) {
  cudaStream_t st = c->setup_stream;
  cublasHandle_t h = c->blas;
  const size_t nn = (size_t)n * n;
  DevBuf a, b, w, info, work, t1, t2;
  a.ensure(sizeof(double) * nn);
  b.ensure(sizeof(double) * nn);
  w.ensure(sizeof(double) * n);
  info.ensure(sizeof(int));
  PE_CUDA_CHECK(cudaMemcpyAsync(a.p, A, sizeof(double) * nn, cudaMemcpyDeviceToDevice, st));
  PE_CUDA_CHECK(cudaMemcpyAsync(b.p, M, sizeof(double) * nn, cudaMemcpyDeviceToDevice, st));
  int lwork = 0;
  SOLVER_CHECK(cusolverDnDsygvd_bufferSize(c->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                           CUBLAS_FILL_MODE_LOWER, n, a.d(), n, b.d(), n, w.d(), &lwork));
  work.ensure(sizeof(double) * std::max(lwork, 1));
  SOLVER_CHECK(cusolverDnDsygvd(c->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                CUBLAS_FILL_MODE_LOWER, n, a.d(), n, b.d(), n, w.d(), work.d(),
                                lwork, info.i()));
  int h_info = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h_info != 0) return false;
  mu.assign(n, 0.0);
  PE_CUDA_CHECK(cudaMemcpyAsync(mu.data(), w.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  // a holds the eigenvectors column-major, i.e. V^T read row-major
  rm_geam(h, true, false, n, n, 1.0, a.d(), n, 0.0, a.d(), n, V, n);
  rm_gemm(h, false, false, n, n, n, 1.0, a.d(), n, M, n, 0.0, Vi, n);
  t1.ensure(sizeof(double) * nn);
  t2.ensure(sizeof(double) * nn);
  rm_gemm(h, false, false, n, n, n, 1.0, A, n, V, n, 0.0, t1.d(), n);          // A V
  rm_gemm(h, false, false, n, n, n, 1.0, a.d(), n, t1.d(), n, 0.0, t2.d(), n);  // V^T A V
  sub_diag_kernel<<<grid_for(n), 256, 0, st>>>(n, t2.d(), n, w.d(), 0.0);
  rm_gemm(h, false, false, n, n, n, 1.0, Vi, n, V, n, 0.0, t1.d(), n);          // V^T M V
  sub_diag_kernel<<<grid_for(n), 256, 0, st>>>(n, t1.d(), n, nullptr, 1.0);
  PE_CUDA_CHECK(cudaGetLastError());
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  double mmax = 0.0;
  for (double x : mu) mmax = std::max(mmax, std::fabs(x));
  const double ep = max_abs(c, (long long)nn, t2.d()), eq = max_abs(c, (long long)nn, t1.d());
  return ep <= 1e-9 * std::max(mmax, 1e-300) && eq <= 1e-9;
}

__global__ void zero_strict_lower_kernel(int n, double* U) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * n;
       t += (long long)gridDim.x * blockDim.x)
    if (t / n > t % n) U[t] = 0.0;
}

// Upper-triangular norm factor: U = L^T with L L^T = V^T V (Cholesky), so ||U e|| = ||V e||
// at half the flops of V e (the residual-norm GEMM skips U's zero k-tiles).
static bool norm_factor(pe_ctx* c, int n, const double* V, double* U) {
  cudaStream_t st = c->setup_stream;
  rm_gemm(c->blas, true, false, n, n, n, 1.0, V, n, V, n, 0.0, U, n);  // V^T V (symmetric)
  DevBuf work, info;
  info.ensure(sizeof(int));
  int lwork = 0;
  SOLVER_CHECK(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, U, n, &lwork));
  work.ensure(sizeof(double) * std::max(lwork, 1));
  SOLVER_CHECK(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, n, U, n, work.d(), lwork, info.i()));
  int h_info = 0;
  PE_CUDA_CHECK(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h_info != 0) return false;
  // column-major lower L read row-major is L^T in the upper triangle; clear the rest
  zero_strict_lower_kernel<<<grid_for((long long)n * n), 256, 0, st>>>(n, U);
  PE_CUDA_CHECK(cudaGetLastError());
  return true;
}

// Operators of the modal WR sweep (wr_modal.cu) for every member; false (and the general
// path is used) unless both pencils pass pencil_eig and every modal time recurrence is
// well posed (1 + mu1 dt > 0, |1 - alpha a^J| >= 1e-6).
static bool setup_modal_full(pe_ctx* c, double dt, double alpha) {
  const int d1 = c->d1, d2 = c->d2, J = c->J, E = c->E;
  if (d1 == 0 || d2 == 0) return false;
  cublasHandle_t h = c->blas;
  cudaStream_t st = c->setup_stream;
  const size_t vstride = (size_t)d1 * d1 + (size_t)d2 * d2;
  c->Vcat.ensure(sizeof(double) * E * vstride + 8);
  c->Vicat.ensure(sizeof(double) * E * vstride + 8);
  c->Ucat.ensure(sizeof(double) * E * vstride + 8);
  c->RT.ensure(sizeof(double) * (size_t)E * d1 * 2 * d2 + 8);
  c->GT.ensure(sizeof(double) * (size_t)E * d2 * 2 * d1 + 8);
  c->f1t.ensure(sizeof(double) * (size_t)E * d1 + 8);
  c->cgt.ensure(sizeof(double) * (size_t)E * d2 + 8);
  c->acoef.ensure(sizeof(double) * (size_t)E * d1 + 8);
  c->cden.ensure(sizeof(double) * (size_t)E * d1 + 8);
  c->lam.ensure(sizeof(double) * (size_t)E * d2 + 8);
  DevBuf t12, t21;
  t12.ensure(sizeof(double) * (size_t)d1 * d2);
  t21.ensure(sizeof(double) * (size_t)d2 * d1);
  std::vector<double> mu1, mu2, ha(d1), hc(d1), hl(d2);
  for (int e = 0; e < E; ++e) {
    const double* M11 = c->M11.d() + (size_t)e * d1 * d1;
    const double* A11 = c->A11.d() + (size_t)e * d1 * d1;
    const double* M12 = c->M12.d() + (size_t)e * d1 * d2;
    const double* A12 = c->A12.d() + (size_t)e * d1 * d2;
    const double* M22 = c->M22.d() + (size_t)e * d2 * d2;
    const double* A22 = c->A22.d() + (size_t)e * d2 * d2;
    double* V1 = c->Vcat.d() + e * vstride;
    double* V2 = V1 + (size_t)d1 * d1;
    double* V1i = c->Vicat.d() + e * vstride;
    double* V2i = V1i + (size_t)d1 * d1;
    if (!pencil_eig(c, d1, A11, M11, V1, V1i, mu1)) return false;
    if (!pencil_eig(c, d2, A22, M22, V2, V2i, mu2)) return false;
    double* U1 = c->Ucat.d() + e * vstride;
    if (!norm_factor(c, d1, V1, U1) || !norm_factor(c, d2, V2, U1 + (size_t)d1 * d1)) return false;
    for (int i = 0; i < d1; ++i) {
      const double q = 1.0 + mu1[i] * dt;
      if (!(q > 0.0)) return false;
      ha[i] = 1.0 / q;
      const double den = 1.0 - alpha * std::pow(ha[i], (double)J);
      if (!(std::fabs(den) >= 1e-6)) return false;
      hc[i] = 1.0 / den;
    }
    for (int i = 0; i < d2; ++i) hl[i] = 1.0 - dt * mu2[i];
    PE_CUDA_CHECK(cudaMemcpyAsync(c->acoef.d() + (size_t)e * d1, ha.data(), 8 * d1, cudaMemcpyHostToDevice, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(c->cden.d() + (size_t)e * d1, hc.data(), 8 * d1, cudaMemcpyHostToDevice, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(c->lam.d() + (size_t)e * d2, hl.data(), 8 * d2, cudaMemcpyHostToDevice, st));
    // V1^T X = (V1^-1 M11^-1) X is not formed: V1^T is read as the transpose of V1
    double* RT = c->RT.d() + (size_t)e * d1 * 2 * d2;
    rm_gemm(h, false, false, d1, d2, d2, 1.0, A12, d2, V2, d2, 0.0, t12.d(), d2);       // A12 V2
    rm_gemm(h, true, false, d1, d2, d1, -1.0, V1, d1, t12.d(), d2, 0.0, RT, 2 * d2);    // -V1^T A12 V2
    rm_gemm(h, false, false, d1, d2, d2, 1.0, M12, d2, V2, d2, 0.0, t12.d(), d2);       // M12 V2
    rm_gemm(h, true, false, d1, d2, d1, -1.0 / dt, V1, d1, t12.d(), d2, 0.0, RT + d2, 2 * d2);
    rm_gemm(h, true, false, d1, 1, d1, 1.0, V1, d1, c->f1.d() + (size_t)e * d1, 1, 0.0,
            c->f1t.d() + (size_t)e * d1, 1);
    double* GT = c->GT.d() + (size_t)e * d2 * 2 * d1;
    rm_gemm(h, true, false, d2, d1, d1, 1.0, A12, d2, V1, d1, 0.0, t21.d(), d1);        // A12^T V1
    rm_gemm(h, true, false, d2, d1, d2, -dt, V2, d2, t21.d(), d1, 0.0, GT, 2 * d1);     // -dt V2^T A12^T V1
    rm_gemm(h, true, false, d2, d1, d1, 1.0, M12, d2, V1, d1, 0.0, t21.d(), d1);        // M12^T V1
    rm_gemm(h, true, false, d2, d1, d2, -1.0, V2, d2, t21.d(), d1, 0.0, GT + d1, 2 * d1);
    rm_gemm(h, true, false, d2, 1, d2, dt, V2, d2, c->f2.d() + (size_t)e * d2, 1, 0.0,
            c->cgt.d() + (size_t)e * d2, 1);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  return true;
}

static void setup_allatonce_general(pe_ctx* c, double dt, double alpha, int npm, bool even);

void setup_allatonce(pe_ctx* c, double dt, double alpha, double tol, int max_iter) {
  const int d1 = c->d1, d2 = c->d2, J = c->J;
  cudaStream_t st = c->setup_stream;
  // Half spectrum in half-complex packing.  The WR right-hand side is real, so
  // Finv[J-k, s] = conj(Finv[k, s]) and d_{J-k} = conj(d_k): Q_{J-k} = conj(Q_k).  Only modes
  // k = 0..floor(J/2) are solved, as npm = ceil(J/2) "pseudo-modes" of two planes each:
  // pseudo-mode 0 carries the real modes k = 0 and (J even) k = J/2, pseudo-mode m >= 1 the
  // re/im planes of mode m.  The transforms are then exactly J (even J) rows deep, and the
  // backward transform weights each conjugate pair by 2.
  const int npm = (J + 1) / 2;
  const bool even = (J % 2) == 0;
  c->wr_nk = npm;
  {
    std::vector<double> finv((size_t)2 * npm * J, 0.0), fw((size_t)J * 2 * npm, 0.0);
    const double two_pi = 6.283185307179586476925286766559;
    auto coef = [&](int k, int s, double& fr, double& fi, double& wr, double& wi) {
      const long long ks = ((long long)k * s) % J;
      const double ang = two_pi * (double)ks / (double)J;
      const double lam_inv = std::pow(alpha, (double)s / J);  // Lambda^{-1}_s
      const double lam = std::pow(alpha, -(double)s / J);     // Lambda_s
      // S^{-1}: p_k = (1/J) sum_s e^{-i ang} alpha^{s/J} r_s
      fr = lam_inv * std::cos(ang) / J;
      fi = -lam_inv * std::sin(ang) / J;
      // Re(S q)_s = sum_k alpha^{-s/J} (cos ang Re q_k - sin ang Im q_k)
      wr = lam * std::cos(ang);
      wi = -lam * std::sin(ang);
    };
    for (int s = 0; s < J; ++s) {
      double fr, fi, wr, wi;
      coef(0, s, fr, fi, wr, wi);  // pseudo-mode 0, plane 0: real mode 0
      finv[(size_t)0 * J + s] = fr;
      fw[(size_t)s * 2 * npm + 0] = wr;
      if (even) {  // plane 1: real mode J/2
        coef(J / 2, s, fr, fi, wr, wi);
        finv[(size_t)1 * J + s] = fr;
        fw[(size_t)s * 2 * npm + 1] = wr;
      }
      for (int m = 1; m < npm; ++m) {
        coef(m, s, fr, fi, wr, wi);
        finv[(size_t)(2 * m) * J + s] = fr;
        finv[(size_t)(2 * m + 1) * J + s] = fi;
        fw[(size_t)s * 2 * npm + 2 * m] = 2.0 * wr;
        fw[(size_t)s * 2 * npm + 2 * m + 1] = 2.0 * wi;
      }
    }
    c->Finv.ensure(sizeof(double) * finv.size());
    c->Fw.ensure(sizeof(double) * fw.size());
    PE_CUDA_CHECK(cudaMemcpy(c->Finv.p, finv.data(), sizeof(double) * finv.size(), cudaMemcpyHostToDevice));
    PE_CUDA_CHECK(cudaMemcpy(c->Fw.p, fw.data(), sizeof(double) * fw.size(), cudaMemcpyHostToDevice));
  }
  // modal sweep when both pencils diagonalise (wr_modal.cu); otherwise the general path
  c->wr_modal = false;
  c->wr_modal_avail = c->use_modal && setup_modal_full(c, dt, alpha);
  c->wr_modal_full = c->wr_modal_avail && !wr_tiny_eligible(d1, d2, J, npm);
  if (!c->wr_modal_full) setup_allatonce_general(c, dt, alpha, npm, even);
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  c->wr_ready = true;
  c->wr_dt = dt;
  c->wr_alpha = alpha;
  c->wr_tol = tol;
  c->wr_max_iter = max_iter;
}

// The general all-at-once operators: shifted inverses, rhs / g operators, E (direct or
// modal w recursion).
static void setup_allatonce_general(pe_ctx* c, double dt, double alpha, int npm, bool even) {
  const int d1 = c->d1, d2 = c->d2, J = c->J, E = c->E;
  cudaStream_t st = c->setup_stream;
  cublasHandle_t h = c->blas;
  c->Bk.ensure(sizeof(double) * (size_t)E * npm * 4 * d1 * d1 + 8);
  c->RW.ensure(sizeof(double) * (size_t)E * d1 * 2 * d2 + 8);
  c->M11dt.ensure(sizeof(double) * (size_t)E * d1 * d1 + 8);
  c->GW.ensure(sizeof(double) * (size_t)E * d2 * 2 * d1 + 8);
  c->cg.ensure(sizeof(double) * (size_t)E * d2 + 8);
  c->Emat.ensure(sizeof(double) * (size_t)E * d2 * d2 + 8);
  // Every member's and every mode's shifted matrix in real block form, inverted in one
  // batched LU pass (batchlu.cu); slot 0 of a member holds the real modes k = 0 and J/2.
  DevBuf S, ipiv, info, M22inv;
  const size_t n2 = 2 * (size_t)d1, per = n2 * n2;
  const int nmat = E * npm;
  if (d1) {
    S.ensure(sizeof(double) * (size_t)nmat * per + 16);
    ipiv.ensure(sizeof(int) * (size_t)nmat * n2 + 16);
    info.ensure(sizeof(int) * (size_t)nmat + 16);
  }
  M22inv.ensure(sizeof(double) * (size_t)d2 * d2 + 8);
  const double om_r = std::pow(alpha, 1.0 / J);
  for (int e = 0; e < E; ++e) {
    const double* M11 = c->M11.d() + (size_t)e * d1 * d1;
    const double* A11 = c->A11.d() + (size_t)e * d1 * d1;
    const double* M12 = c->M12.d() + (size_t)e * d1 * d2;
    const double* A12 = c->A12.d() + (size_t)e * d1 * d2;
    const double* M22 = c->M22.d() + (size_t)e * d2 * d2;
    const double* A22 = c->A22.d() + (size_t)e * d2 * d2;
    const double* f2 = c->f2.d() + (size_t)e * d2;
    if (d1) {
      double* S0 = S.d() + (size_t)e * npm * per;
      PE_CUDA_CHECK(cudaMemsetAsync(S0, 0, sizeof(double) * per, st));
      if (!even)
        shifted_real_block_kernel<<<grid_for((long long)d1 * d1), 256, 0, st>>>(
            d1, 0.0, M11, A11, S0, 1, 1);
      for (int k = 0; k <= J / 2; ++k) {
        // d_k = (1 - alpha^{1/J} e^{-2 pi i k/J}) / dt   (allatonce.py:58-62)
        const double ang = -6.283185307179586476925286766559 * (double)k / J;
        const double dre = (1.0 - om_r * std::cos(ang)) / dt;
        const double dim = (-om_r * std::sin(ang)) / dt;
        if (k == 0 || (even && 2 * k == J))  // real modes: diagonal block of pseudo-mode 0
          shifted_real_block_kernel<<<grid_for((long long)d1 * d1), 256, 0, st>>>(
              d1, dre, M11, A11, S0, k == 0 ? 0 : 1, 0);
        else
          shifted_blockform_kernel<<<grid_for((long long)d1 * d1), 256, 0, st>>>(
              d1, dre, dim, M11, A11, S0 + (size_t)k * per);
        PE_CUDA_CHECK(cudaGetLastError());
      }
      double* RW = c->RW.d() + (size_t)e * d1 * 2 * d2;
      // [-A12 | -M12/dt] acting on [w_{s}; w_{s} - w_{s-1}]: difference first, like
      // build_rhs's dw = (w_hist[1:] - w_hist[:-1]) / dt (allatonce.py:154-156)
      rm_geam(h, false, false, d1, d2, -1.0, A12, d2, 0.0, A12, d2, RW, 2 * d2);
      rm_geam(h, false, false, d1, d2, -1.0 / dt, M12, d2, 0.0, M12, d2, RW + d2, 2 * d2);
      rm_geam(h, false, false, d1, d1, 1.0 / dt, M11, d1, 0.0, M11, d1,
              c->M11dt.d() + (size_t)e * d1 * d1, d1);
    }
    if (d2) {
      inverse(c, d2, M22, M22inv.d());
      double* Em = c->Emat.d() + (size_t)e * d2 * d2;
      set_identity(d2, Em, d2, 1.0, st);
      rm_gemm(h, false, false, d2, d2, d2, -dt, M22inv.d(), d2, A22, d2, 1.0, Em, d2);
      // g = dt M22inv^T (f2 - M12^T du/dt - A12^T u)   (row form `@ m22_inv`, :224)
      rm_gemm(h, true, false, d2, 1, d2, dt, M22inv.d(), d2, f2, 1, 0.0,
              c->cg.d() + (size_t)e * d2, 1);
      if (d1) {
        double* GW = c->GW.d() + (size_t)e * d2 * 2 * d1;
        rm_gemm(h, true, true, d2, d1, d2, -dt, M22inv.d(), d2, A12, d2, 0.0, GW, 2 * d1);
        rm_gemm(h, true, true, d2, d1, d2, -1.0, M22inv.d(), d2, M12, d2, 0.0, GW + d1, 2 * d1);
      }
    }
  }
  if (d1) {
    batched_lu_inverse((int)n2, nmat, S.d(), c->Bk.d(), ipiv.i(), info.i(), st);
    if (!even)
      for (int e = 0; e < E; ++e)
        clear_block_kernel<<<grid_for((long long)d1 * d1), 256, 0, st>>>(
            d1, c->Bk.d() + (size_t)e * npm * per, 1);
    // one host round trip for every mode's factorisation status
    std::vector<int> h_info((size_t)nmat);
    PE_CUDA_CHECK(cudaMemcpyAsync(h_info.data(), info.p, sizeof(int) * h_info.size(),
                                  cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    for (size_t q = 0; q < h_info.size(); ++q)
      if (h_info[q] != 0)
        throw Error{PE_ERR_SOLVER, "singular shifted matrix d_k M11 + A11 (member " +
                                       std::to_string(q / npm) + ", pseudo-mode " +
                                       std::to_string(q % npm) + ", zero pivot " +
                                       std::to_string(h_info[q]) + ")"};
  }
  if (wr_tiny_eligible(d1, d2, J, npm)) {  // transposed Bk for the fused small-problem path
    c->BkT.ensure(sizeof(double) * (size_t)E * npm * 4 * d1 * d1 + 8);
    transpose_blocks(E * npm, 2 * d1, c->Bk.d(), c->BkT.d(), st);
  }
  if (c->use_modal && d2 > 0 && !wr_tiny_eligible(d1, d2, J, npm)) {
    c->Vm.ensure(sizeof(double) * (size_t)E * d2 * d2 + 8);
    c->Vinv.ensure(sizeof(double) * (size_t)E * d2 * d2 + 8);
    c->lam.ensure(sizeof(double) * (size_t)E * d2 + 8);
    c->GZ.ensure(sizeof(double) * (size_t)E * d2 * 2 * d1 + 8);
    c->cgz.ensure(sizeof(double) * (size_t)E * d2 + 8);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    bool ok = true;
    for (int e = 0; e < E && ok; ++e)
      ok = setup_modal(c, e, dt, c->M22.d() + (size_t)e * d2 * d2, c->A22.d() + (size_t)e * d2 * d2,
                       c->Emat.d() + (size_t)e * d2 * d2, c->GW.d() + (size_t)e * d2 * 2 * d1,
                       c->cg.d() + (size_t)e * d2);
    c->wr_modal = ok;
  }
}

}  // namespace pe
