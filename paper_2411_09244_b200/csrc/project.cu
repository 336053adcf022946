// Galerkin projection of the fine operators onto the split multiscale basis (SURVEY §8f
// row 1, the projection part of the offline build): msbasis.py:545-567 project_coarse
// (Psi_i^T X Psi_j for X in {M, A}, diagonal blocks symmetrised) and msbasis.py:570-572
// project_load (Psi^T b).
//
// The basis arrives as host CSR of P = [Psi1 Psi2] (n x d).  It is expanded once to a
// dense column-major Psi (leading dimension ldp = n rounded up to 32, zero rows below n),
// Y = X Psi is a CSR SpMM (one thread per (row, column), coalesced over rows), and
// Psi^T Y is one FP64 DMMA GEMM (gemm_f64) with K = ldp; the zero rows add exact zeros.

#include <cmath>
#include <string>

#include "pe.h"
#include "pe_internal.h"

namespace pe {

extern long long g_launches;

namespace {

template <class T>
struct DevP {
  T* p = nullptr;
  explicit DevP(size_t n) {
    if (n) {
      cudaError_t e = cudaMalloc(&p, n * sizeof(T));
      if (e != cudaSuccess)
        throw Error{PE_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
    }
  }
  ~DevP() { cudaFree(p); }
  DevP(const DevP&) = delete;
  DevP& operator=(const DevP&) = delete;
};

template <class T>
void up(T* d, const T* h, size_t n, cudaStream_t st) {
  if (n) PE_CUDA_CHECK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

__global__ void k_expand_basis(int n, long long ldp, const int* __restrict__ pp,
                               const int* __restrict__ pi, const double* __restrict__ pv,
                               double* __restrict__ Psi) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int t = pp[i]; t < pp[i + 1]; ++t) Psi[(long long)pi[t] * ldp + i] = pv[t];
}

// Y(:, j) = X Psi(:, j); grid.y walks the columns.
__global__ void k_spmm_cols(int n, long long ldp, int d, const int* __restrict__ xp,
                            const int* __restrict__ xi, const double* __restrict__ xv,
                            const double* __restrict__ Psi, double* __restrict__ Y) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = blockIdx.y; j < d; j += gridDim.y) {
    const double* pj = Psi + (long long)j * ldp;
    double s = 0.0;
    for (int t = xp[i]; t < xp[i + 1]; ++t) s = fma(xv[t], pj[xi[t]], s);
    Y[(long long)j * ldp + i] = s;
  }
}

// out (row-major d x d) from C (row-major d x d): diagonal blocks (b + b^T) / 2 with the
// removed asymmetry max |b - b^T| reduced per CTA into asym[blockIdx] (max is exact).
__global__ void k_symmetrise(int d, int d1, const double* __restrict__ C, double* __restrict__ O,
                             double* __restrict__ asym) {
  __shared__ double red[256];
  double m = 0.0;
  long long tot = (long long)d * d;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    int i = (int)(t / d), j = (int)(t % d);
    bool diag = (i < d1) == (j < d1);
    double c = C[t];
    if (diag) {
      double ct = C[(long long)j * d + i];
      m = fmax(m, fabs(c - ct));
      O[t] = (c + ct) / 2;
    } else {
      O[t] = c;
    }
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) asym[blockIdx.x] = red[0];
}

// f(j) = Psi(:, j)^T b, one warp per column, fixed-order shuffle sum.
__global__ void k_basis_dot(int n, long long ldp, int d, const double* __restrict__ Psi,
                            const double* __restrict__ b, double* __restrict__ f) {
  int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= d) return;
  const double* pj = Psi + (long long)j * ldp;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s = fma(pj[i], b[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) f[j] = s;
}

// f(j) = sum_t val[t] b[row[t]] over column j of a CSC matrix: one warp per column,
// lane-strided partial sums combined in a fixed xor-shuffle order (deterministic).
__global__ void k_csc_dot(int d, const int* __restrict__ cp, const int* __restrict__ ci,
                          const double* __restrict__ cv, const double* __restrict__ b,
                          double* __restrict__ f) {
  int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= d) return;
  double s = 0.0;
  for (int t = cp[j] + lane; t < cp[j + 1]; t += 32) s = fma(cv[t], b[ci[t]], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) f[j] = s;
}

}  // namespace

static void project_load_impl(int n, int d, const int* cp_h, const int* ci_h, const double* cv_h,
                              const double* b_h, double* f_h, cudaStream_t st) {
  const int nnz = cp_h[d];
  DevP<int> cp(d + 1), ci(nnz);
  DevP<double> cv(nnz), b(n), f(d);
  up(cp.p, cp_h, d + 1, st);
  up(ci.p, ci_h, nnz, st);
  up(cv.p, cv_h, nnz, st);
  up(b.p, b_h, n, st);
  k_csc_dot<<<(d + 7) / 8, 256, 0, st>>>(d, cp.p, ci.p, cv.p, b.p, f.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  PE_CUDA_CHECK(cudaMemcpyAsync(f_h, f.p, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
}

struct ProjArgs {
  int n, d1, d2, nx;
  const int *pp, *pi;
  const double* pv;
  const int* const* xp;
  const int* const* xi;
  const double* const* xv;
  const double* b;
  double** out;
  double* asym_h;
  double* f_h;
  cudaStream_t st;
};

static void project_impl(ProjArgs& a) {
  const int n = a.n, d = a.d1 + a.d2;
  const long long ldp = ((long long)n + 31) & ~31LL;
  const int nnz_p = a.pp[n];
  DevP<int> pp(n + 1), pi(nnz_p);
  DevP<double> pv(nnz_p), Psi((size_t)ldp * d), Y((size_t)ldp * d), C((size_t)d * d),
      O((size_t)d * d);
  const int nred = 148;
  DevP<double> asym(nred);
  up(pp.p, a.pp, n + 1, a.st);
  up(pi.p, a.pi, nnz_p, a.st);
  up(pv.p, a.pv, nnz_p, a.st);
  PE_CUDA_CHECK(cudaMemsetAsync(Psi.p, 0, sizeof(double) * ldp * d, a.st));
  PE_CUDA_CHECK(cudaMemsetAsync(Y.p, 0, sizeof(double) * ldp * d, a.st));
  k_expand_basis<<<(n + 255) / 256, 256, 0, a.st>>>(n, ldp, pp.p, pi.p, pv.p, Psi.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  for (int x = 0; x < a.nx; ++x) {
    const int nnz = a.xp[x][n];
    DevP<int> xp(n + 1), xi(nnz);
    DevP<double> xv(nnz);
    up(xp.p, a.xp[x], n + 1, a.st);
    up(xi.p, a.xi[x], nnz, a.st);
    up(xv.p, a.xv[x], nnz, a.st);
    dim3 g((n + 255) / 256, d < 1024 ? d : 1024);
    k_spmm_cols<<<g, 256, 0, a.st>>>(n, ldp, d, xp.p, xi.p, xv.p, Psi.p, Y.p);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
    GemmParams p;
    p.M = d;
    p.N = d;
    p.nseg = 1;
    p.seg[0].A = Operand{Psi.p, ldp, 1, 0, 0};
    p.seg[0].B = Operand{Y.p, 1, ldp, 0, 0};
    p.seg[0].K = (int)ldp;
    p.C = C.p;
    p.c_i = d;
    p.c_j = 1;
    gemm_f64(p, a.st);
    k_symmetrise<<<nred, 256, 0, a.st>>>(d, a.d1, C.p, O.p, asym.p);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
    double red[nred];
    PE_CUDA_CHECK(cudaMemcpyAsync(red, asym.p, sizeof(red), cudaMemcpyDeviceToHost, a.st));
    PE_CUDA_CHECK(cudaMemcpyAsync(a.out[x], O.p, sizeof(double) * d * d, cudaMemcpyDeviceToHost,
                                  a.st));
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
    double m = 0.0;
    for (int i = 0; i < nred; ++i) m = std::fmax(m, red[i]);
    if (a.asym_h) a.asym_h[x] = m;
  }
  if (a.b && a.f_h) {
    DevP<double> b(n), f(d);
    up(b.p, a.b, n, a.st);
    k_basis_dot<<<(d + 7) / 8, 256, 0, a.st>>>(n, ldp, d, Psi.p, b.p, f.p);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
    PE_CUDA_CHECK(cudaMemcpyAsync(a.f_h, f.p, sizeof(double) * d, cudaMemcpyDeviceToHost, a.st));
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
  }
}

}  // namespace pe

extern "C" int pe_project_coarse(int n, int d1, int d2, const int* P_ptr, const int* P_idx,
                                 const double* P_val, const int* M_ptr, const int* M_idx,
                                 const double* M_val, const int* A_ptr, const int* A_idx,
                                 const double* A_val, const double* b, double* Mc_h,
                                 double* Ac_h, double* f_h, double* asym_h, void* stream) {
  if (n <= 0 || d1 < 0 || d2 < 0 || d1 + d2 <= 0 || !P_ptr || !M_ptr || !A_ptr || !Mc_h ||
      !Ac_h) {
    pe::set_error("pe_project_coarse: need n > 0, d1 + d2 > 0 and buffers");
    return PE_ERR_ARG;
  }
  const int* xp[2] = {M_ptr, A_ptr};
  const int* xi[2] = {M_idx, A_idx};
  const double* xv[2] = {M_val, A_val};
  double* out[2] = {Mc_h, Ac_h};
  pe::ProjArgs a{n, d1, d2, 2, P_ptr, P_idx, P_val, xp, xi, xv, b, out, asym_h, f_h,
                 (cudaStream_t)stream};
  try {
    pe::project_impl(a);
    return PE_OK;
  } catch (const pe::Error& e) {
    pe::set_error("pe_project_coarse: " + e.msg);
    return e.code;
  } catch (const std::exception& e) {
    pe::set_error(std::string("pe_project_coarse: ") + e.what());
    return PE_ERR_CUDA;
  }
}

extern "C" int pe_project_load(int n, int d, const int* P_colptr, const int* P_rowidx,
                               const double* P_val, const double* b, double* f_h, void* stream) {
  if (n <= 0 || d <= 0 || !P_colptr || !b || !f_h || (P_colptr[d] > 0 && (!P_rowidx || !P_val))) {
    pe::set_error("pe_project_load: need n > 0, d > 0 and buffers");
    return PE_ERR_ARG;
  }
  for (int j = 0; j < d; ++j)
    if (P_colptr[j + 1] < P_colptr[j]) {
      pe::set_error("pe_project_load: column pointers must be non-decreasing");
      return PE_ERR_ARG;
    }
  for (int t = 0; t < P_colptr[d]; ++t)
    if (P_rowidx[t] < 0 || P_rowidx[t] >= n) {
      pe::set_error("pe_project_load: row index out of range");
      return PE_ERR_ARG;
    }
  try {
    pe::project_load_impl(n, d, P_colptr, P_rowidx, P_val, b, f_h, (cudaStream_t)stream);
    return PE_OK;
  } catch (const pe::Error& e) {
    pe::set_error("pe_project_load: " + e.msg);
    return e.code;
  } catch (const std::exception& e) {
    pe::set_error(std::string("pe_project_load: ") + e.what());
    return PE_ERR_CUDA;
  }
}
