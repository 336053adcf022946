// CEM-GMsFEM multiscale basis on the GPU (the offline build):
// msbasis.py:296-328 aux_eigen_cem and :331-394 build_cem_basis for every coarse block of a
// uniform nx x nx Q1 grid cut into nb x nb blocks.
//
//  1. Auxiliary spectral problems, all blocks batched: on block b's free nodes (the block
//     rectangle's nodes minus the global Dirichlet boundary; natural on the block edges)
//       a(psi, v) = lambda s(psi, v),  a = sum_cells kappa K_ref,  s = sum_cells kt h^2 M_ref,
//     kt = kappa nb^2 (the "kappa_h2" weight, msbasis.py:266-268).  Dense per block, padded
//     to (s+1)^2 with a decoupled (I, I) block: S = L L^T (batched potrf),
//     C = L^-1 A L^-T (batched trsm; the padded diagonal then set just above a Gershgorin
//     bound of the real part, so the padding sorts last without inflating ||C||),
//     C = Y diag(w) Y^T (batched syev, ascending), V = L^-T Y
//     (s-orthonormal), the first n_eig columns with the reference's sign (largest-magnitude
//     entry positive, first such entry).
//  2. Constraint functions W_j = s_j V_j on each block's free nodes (batched GEMM).
//  3. Per block b, the energy minimisation on its oversampled patch (patch-interior nodes,
//     zero Dirichlet rim): min a(phi, phi) subject to C phi = e_t, with the rows of C the
//     restrictions of W_j (j over the patch blocks, ascending, n_eig each).  The KKT system
//     [[A, C^T], [C, 0]] (solved by sparse LU in the reference) is solved by its Schur
//     complement: A = L L^T, Y = A^-1 C^T, G = C Y, phi = Y G^-1 E_t for the n_eig targets,
//     then two steps of iterative refinement on the full KKT system.  Dense per block (patch
//     <= 55^2 nodes at config 3), cuSOLVER potrf / potrs.
//
// Output: per block, the n_eig basis columns on its patch-interior nodes (row-major
// node order), plus the worst constraint residual |C phi - e|.

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "pe.h"
#include "pe_internal.h"

namespace pe {

extern long long g_launches;

namespace {

__constant__ double kStiff[16] = {4.0 / 6, -1.0 / 6, -2.0 / 6, -1.0 / 6,   //
                                  -1.0 / 6, 4.0 / 6, -1.0 / 6, -2.0 / 6,   //
                                  -2.0 / 6, -1.0 / 6, 4.0 / 6, -1.0 / 6,   //
                                  -1.0 / 6, -2.0 / 6, -1.0 / 6, 4.0 / 6};
__constant__ double kMass[16] = {4.0 / 36, 2.0 / 36, 1.0 / 36, 2.0 / 36,  //
                                 2.0 / 36, 4.0 / 36, 2.0 / 36, 1.0 / 36,  //
                                 1.0 / 36, 2.0 / 36, 4.0 / 36, 2.0 / 36,  //
                                 2.0 / 36, 1.0 / 36, 2.0 / 36, 4.0 / 36};

// local index (SW 0, SE 1, NE 2, NW 3) of node (x, y) in cell (cx, cy), or -1
__device__ __forceinline__ int corner(int x, int y, int cx, int cy) {
  const int dx = x - cx, dy = y - cy;
  if (dx < 0 || dx > 1 || dy < 0 || dy > 1) return -1;
  return dy == 0 ? dx : 3 - dx;
}

// sum over the cells of [cx0, cx1) x [cy0, cy1) that contain both nodes p and q of
// w_c * ref[lp][lq] (cells visited in ascending (cy, cx) order)
template <bool STIFF>
__device__ double pair_sum(int px, int py, int qx, int qy, int cx0, int cx1, int cy0, int cy1,
                           int nx, const double* __restrict__ wcell) {
  double s = 0.0;
  const int ylo = max(max(py, qy) - 1, cy0), yhi = min(min(py, qy), cy1 - 1);
  const int xlo = max(max(px, qx) - 1, cx0), xhi = min(min(px, qx), cx1 - 1);
  for (int cy = ylo; cy <= yhi; ++cy)
    for (int cx = xlo; cx <= xhi; ++cx) {
      const int lp = corner(px, py, cx, cy), lq = corner(qx, qy, cx, cy);
      if (lp < 0 || lq < 0) continue;
      const double ref = STIFF ? kStiff[lp * 4 + lq] : kMass[lp * 4 + lq];
      s = fma(wcell[(long long)cy * nx + cx], ref, s);
    }
  return s;
}

struct CemGeom {
  int nx, nb, s, layers, n;  // n = (s + 1)^2 padded block size
};

// free node list of block b (ascending node order) -> (x, y) of local index i, or false
__device__ __forceinline__ bool block_free_node(const CemGeom& g, int b, int i, int* x, int* y) {
  const int bx = b % g.nb, by = b / g.nb;
  int k = 0;
  for (int yy = by * g.s; yy <= (by + 1) * g.s; ++yy) {
    if (yy == 0 || yy == g.nx) continue;
    const int xlo = bx * g.s, xhi = (bx + 1) * g.s;
    const int xa = max(xlo, 1), xb = min(xhi, g.nx - 1);
    const int cnt = xb >= xa ? xb - xa + 1 : 0;
    if (i < k + cnt) {
      *x = xa + (i - k);
      *y = yy;
      return true;
    }
    k += cnt;
  }
  return false;
}

__device__ __forceinline__ int block_free_count(const CemGeom& g, int b) {
  const int bx = b % g.nb, by = b / g.nb;
  const int xa = max(bx * g.s, 1), xb = min((bx + 1) * g.s, g.nx - 1);
  const int ya = max(by * g.s, 1), yb = min((by + 1) * g.s, g.nx - 1);
  return (xb - xa + 1) * (yb - ya + 1);
}

// aux matrices, column-major n x n per block: A (stiffness on block cells), S (kt-weighted
// mass), padded rows / columns: A = pad I, S = I
__global__ void k_aux_assemble(CemGeom g, const double* __restrict__ kappa,
                               const double* __restrict__ kt, double pad, double* A, double* S,
                               double* S_keep) {
  const int b = blockIdx.y;
  const int n = g.n;
  const int nf = block_free_count(g, b);
  const int bx = b % g.nb, by = b / g.nb;
  const int cx0 = bx * g.s, cx1 = cx0 + g.s, cy0 = by * g.s, cy1 = cy0 + g.s;
  const double h2 = 1.0 / ((double)g.nx * g.nx);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * n; t += gridDim.x * blockDim.x) {
    const int i = t % n, j = t / n;  // column-major (i row, j column)
    double a = 0.0, m = 0.0;
    if (i < nf && j < nf) {
      int px, py, qx, qy;
      block_free_node(g, b, i, &px, &py);
      block_free_node(g, b, j, &qx, &qy);
      if (abs(px - qx) <= 1 && abs(py - qy) <= 1) {
        a = pair_sum<true>(px, py, qx, qy, cx0, cx1, cy0, cy1, g.nx, kappa);
        m = pair_sum<false>(px, py, qx, qy, cx0, cx1, cy0, cy1, g.nx, kt) * h2;
      }
    } else if (i == j) {
      a = pad;
      m = 1.0;
    }
    const long long o = (long long)b * n * n + t;
    A[o] = a;
    S[o] = m;
    S_keep[o] = m;
  }
}

// After the reduction C = L^-1 A L^-T: the padded (decoupled) diagonal is set just above a
// Gershgorin bound of the block's real part, so the padded eigenvalues sort after every real
// one while ||C|| -- and with it the eigensolver's absolute error -- stays at the real scale.
__global__ void k_aux_pad(CemGeom g, double* C) {
  const int b = blockIdx.x, n = g.n, nf = block_free_count(g, b);
  double* c = C + (long long)b * n * n;
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < nf; i += blockDim.x) {
    double r = 0.0;
    for (int j = 0; j < nf; ++j) r += fabs(c[(long long)j * n + i]);
    m = fmax(m, r);
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const double pad = 2.0 * red[0] + 1.0;
  for (int i = nf + threadIdx.x; i < n; i += blockDim.x) c[(long long)i * n + i] = pad;
}

// sign convention (msbasis.py:321-324): per column k < n_eig, the first entry of largest
// magnitude over the free rows is made positive.  One warp per (block, column).
__global__ void k_aux_sign(CemGeom g, int n_eig, double* V) {
  const int b = blockIdx.x, k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= n_eig) return;
  const int n = g.n, nf = block_free_count(g, b);
  double* col = V + (long long)b * n * n + (long long)k * n;
  double best = -1.0;
  int arg = 0;
  for (int i = lane; i < nf; i += 32) {
    const double a = fabs(col[i]);
    if (a > best) {
      best = a;
      arg = i;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) {
      best = ob;
      arg = oa;
    }
  }
  const bool flip = col[arg] < 0.0;
  __syncwarp();
  if (flip)
    for (int i = lane; i < nf; i += 32) col[i] = -col[i];
}

// patch geometry of block b: interior node rectangle [x0, x1] x [y0, y1] (inclusive)
struct Patch {
  int x0, x1, y0, y1, nxl, n, jb0x, jb1x, jb0y, jb1y;
};
__host__ __device__ inline Patch patch_of(const CemGeom& g, int b) {
  const int bx = b % g.nb, by = b / g.nb;
  Patch p;
  p.jb0x = std::max(bx - g.layers, 0);
  p.jb1x = std::min(bx + g.layers + 1, g.nb);
  p.jb0y = std::max(by - g.layers, 0);
  p.jb1y = std::min(by + g.layers + 1, g.nb);
  p.x0 = p.jb0x * g.s + 1;
  p.x1 = p.jb1x * g.s - 1;
  p.y0 = p.jb0y * g.s + 1;
  p.y1 = p.jb1y * g.s - 1;
  p.nxl = p.x1 - p.x0 + 1;
  p.n = p.nxl * (p.y1 - p.y0 + 1);
  return p;
}

// dense patch stiffness (column-major nl x nl), full-grid stiffness restricted to the patch
// interior nodes (msbasis.py:189-190)
__global__ void k_patch_stiffness(CemGeom g, Patch pt, const double* __restrict__ kappa,
                                  double* A) {
  const long long nl = pt.n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl * nl;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % nl), j = (int)(t / nl);
    const int px = pt.x0 + i % pt.nxl, py = pt.y0 + i / pt.nxl;
    const int qx = pt.x0 + j % pt.nxl, qy = pt.y0 + j / pt.nxl;
    double a = 0.0;
    if (abs(px - qx) <= 1 && abs(py - qy) <= 1)
      a = pair_sum<true>(px, py, qx, qy, 0, g.nx, 0, g.nx, g.nx, kappa);
    A[t] = a;
  }
}

// C^T (column-major nl x m): column r = (patch block j in ascending order, aux k) holds
// W_j[:, k] at the patch-interior nodes that are free nodes of block j
__global__ void k_constraints(CemGeom g, Patch pt, int n_eig, const double* __restrict__ W,
                              double* Ct) {
  const int nbx = pt.jb1x - pt.jb0x;
  const int r = blockIdx.y;  // row of C
  const int q = r / n_eig, k = r % n_eig;
  const int jb = (pt.jb0y + q / nbx) * g.nb + pt.jb0x + q % nbx;
  const int jbx = jb % g.nb, jby = jb / g.nb;
  const int nfx0 = std::max(jbx * g.s, 1), nfx1 = std::min((jbx + 1) * g.s, g.nx - 1);
  const int nfy0 = std::max(jby * g.s, 1);
  const int nfw = nfx1 - nfx0 + 1;
  double* col = Ct + (long long)r * pt.n;
  const double* wj = W + (long long)jb * g.n * n_eig + (long long)k * g.n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pt.n; i += gridDim.x * blockDim.x) {
    const int px = pt.x0 + i % pt.nxl, py = pt.y0 + i / pt.nxl;
    double v = 0.0;
    if (px >= jbx * g.s && px <= (jbx + 1) * g.s && py >= jby * g.s && py <= (jby + 1) * g.s)
      v = wj[(py - nfy0) * nfw + (px - nfx0)];
    col[i] = v;
  }
}

template <class T>
struct Dv {
  T* p = nullptr;
  size_t n = 0;
  explicit Dv(size_t cnt = 0) { alloc(cnt); }
  void alloc(size_t cnt) {
    if (cnt <= n) return;
    cudaFree(p);
    p = nullptr;
    n = 0;
    if (cnt && cudaMalloc(&p, cnt * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error{PE_ERR_NOMEM, "cudaMalloc failed in the CEM build"};
    }
    n = cnt;
  }
  ~Dv() { cudaFree(p); }
  Dv(const Dv&) = delete;
  Dv& operator=(const Dv&) = delete;
};

#define CEM_SOLVER(x)                                                                 \
  do {                                                                                \
    cusolverStatus_t _s = (x);                                                        \
    if (_s != CUSOLVER_STATUS_SUCCESS)                                                \
      throw Error{PE_ERR_SOLVER, std::string(#x) + " failed: " + std::to_string(_s)}; \
  } while (0)
#define CEM_BLAS(x)                                                                   \
  do {                                                                                \
    cublasStatus_t _s = (x);                                                          \
    if (_s != CUBLAS_STATUS_SUCCESS)                                                  \
      throw Error{PE_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(_s)};   \
  } while (0)

int grid_for(long long n, int threads) {
  return (int)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 148LL * 16));
}

}  // namespace

struct CemArgs {
  int nx, nb, layers, n_eig;
  const double* kappa;  // host, nx * nx cells (row-major, cell (cx, cy) at cy * nx + cx)
  double kt_scale;      // kt = kappa * kt_scale (kappa_h2: nb^2)
  double* values;       // host out: per block, n_eig columns of its patch-interior values
  long long* offsets;   // host out: (nb^2 + 1) offsets into values
  double* eigenvalues;  // host out (optional): nb^2 x n_eig aux eigenvalues
  double* worst;        // host out (optional): worst constraint residual
  cudaStream_t st;
};

static void cem_impl(CemArgs& a) {
  CemGeom g;
  g.nx = a.nx;
  g.nb = a.nb;
  g.s = a.nx / a.nb;
  g.layers = a.layers;
  g.n = (g.s + 1) * (g.s + 1);
  const int nblk = a.nb * a.nb, n = g.n, ne = a.n_eig;
  cudaStream_t st = a.st;
  cusolverDnHandle_t sol = nullptr;
  cublasHandle_t bl = nullptr;
  CEM_SOLVER(cusolverDnCreate(&sol));
  struct HS {
    cusolverDnHandle_t s;
    cublasHandle_t b;
    ~HS() {
      if (s) cusolverDnDestroy(s);
      if (b) cublasDestroy(b);
    }
  } hs{sol, nullptr};
  CEM_BLAS(cublasCreate(&bl));
  hs.b = bl;
  CEM_SOLVER(cusolverDnSetStream(sol, st));
  CEM_BLAS(cublasSetStream(bl, st));

  const size_t cells = (size_t)a.nx * a.nx;
  Dv<double> kap(cells), kt(cells);
  {
    std::vector<double> h(a.kappa, a.kappa + cells), w(cells);
    for (size_t c = 0; c < cells; ++c) w[c] = h[c] * a.kt_scale;
    PE_CUDA_CHECK(cudaMemcpyAsync(kap.p, h.data(), cells * 8, cudaMemcpyHostToDevice, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(kt.p, w.data(), cells * 8, cudaMemcpyHostToDevice, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  // ---- 1. aux eigenproblems, batched over blocks
  const size_t nn = (size_t)n * n;
  Dv<double> W((size_t)nblk * n * ne), ev((size_t)nblk * n);
  const double one = 1.0, zero = 0.0;
  {  // aux work buffers (freed before the patch solves)
  Dv<double> A(nn * nblk), S(nn * nblk), Sk(nn * nblk);
  const double pad = 1.0;  // placeholder; k_aux_pad sets the padded eigenvalues after reduction
  k_aux_assemble<<<dim3(std::max(1, std::min(64, (int)((nn + 255) / 256))), nblk), 256, 0, st>>>(
      g, kap.p, kt.p, pad, A.p, S.p, Sk.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  std::vector<double*> hA(nblk), hS(nblk);
  for (int b = 0; b < nblk; ++b) {
    hA[b] = A.p + nn * b;
    hS[b] = S.p + nn * b;
  }
  Dv<double*> dA(nblk), dS(nblk);
  Dv<int> info(nblk + 8);
  PE_CUDA_CHECK(cudaMemcpyAsync(dA.p, hA.data(), nblk * sizeof(double*), cudaMemcpyHostToDevice, st));
  PE_CUDA_CHECK(cudaMemcpyAsync(dS.p, hS.data(), nblk * sizeof(double*), cudaMemcpyHostToDevice, st));
  CEM_SOLVER(cusolverDnDpotrfBatched(sol, CUBLAS_FILL_MODE_LOWER, n, dS.p, n, info.p, nblk));
  {
    std::vector<int> hi(nblk);
    PE_CUDA_CHECK(cudaMemcpyAsync(hi.data(), info.p, nblk * sizeof(int), cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int b = 0; b < nblk; ++b)
      if (hi[b] != 0)
        throw Error{PE_ERR_SOLVER, "aux mass matrix not positive definite on block " + std::to_string(b)};
  }
  // C = L^-1 A L^-T
  CEM_BLAS(cublasDtrsmBatched(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                              CUBLAS_DIAG_NON_UNIT, n, n, &one, dS.p, n, dA.p, n, nblk));
  CEM_BLAS(cublasDtrsmBatched(bl, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                              CUBLAS_DIAG_NON_UNIT, n, n, &one, dS.p, n, dA.p, n, nblk));
  k_aux_pad<<<nblk, 256, 0, st>>>(g, A.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  {
    cusolverDnParams_t prm;
    CEM_SOLVER(cusolverDnCreateParams(&prm));
    size_t wd = 0, wh = 0;
    CEM_SOLVER(cusolverDnXsyevBatched_bufferSize(sol, prm, CUSOLVER_EIG_MODE_VECTOR,
                                                 CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A.p, n,
                                                 CUDA_R_64F, ev.p, CUDA_R_64F, &wd, &wh, nblk));
    Dv<char> work(std::max<size_t>(wd, 1));
    std::vector<char> hwork(std::max<size_t>(wh, 1));
    CEM_SOLVER(cusolverDnXsyevBatched(sol, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                      CUDA_R_64F, A.p, n, CUDA_R_64F, ev.p, CUDA_R_64F, work.p,
                                      wd, hwork.data(), wh, info.p, nblk));
    std::vector<int> hi(nblk);
    PE_CUDA_CHECK(cudaMemcpyAsync(hi.data(), info.p, nblk * sizeof(int), cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    cusolverDnDestroyParams(prm);
    for (int b = 0; b < nblk; ++b)
      if (hi[b] != 0)
        throw Error{PE_ERR_SOLVER, "aux eigensolve failed on block " + std::to_string(b)};
  }
  // V = L^-T Y
  CEM_BLAS(cublasDtrsmBatched(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                              CUBLAS_DIAG_NON_UNIT, n, n, &one, dS.p, n, dA.p, n, nblk));
  k_aux_sign<<<nblk, 32 * ne, 0, st>>>(g, ne, A.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  // ---- 2. W_b = s_b V_b[:, :n_eig]  (n x ne per block, column-major)
  CEM_BLAS(cublasDgemmStridedBatched(bl, CUBLAS_OP_N, CUBLAS_OP_N, n, ne, n, &one, Sk.p, n, nn,
                                     A.p, n, nn, &zero, W.p, n, (long long)n * ne, nblk));
  if (a.eigenvalues) {
    std::vector<double> h((size_t)nblk * n);
    PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), ev.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int b = 0; b < nblk; ++b)
      for (int k = 0; k < ne; ++k) a.eigenvalues[(size_t)b * ne + k] = h[(size_t)b * n + k];
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  }

  // ---- 3. saddle-point solve per block
  a.offsets[0] = 0;
  for (int b = 0; b < nblk; ++b) a.offsets[b + 1] = a.offsets[b] + (long long)patch_of(g, b).n * ne;
  int nl_max = 0, m_max = 0;
  for (int b = 0; b < nblk; ++b) {
    const Patch p = patch_of(g, b);
    nl_max = std::max(nl_max, p.n);
    m_max = std::max(m_max, (p.jb1x - p.jb0x) * (p.jb1y - p.jb0y) * ne);
  }
  Dv<double> Al((size_t)nl_max * nl_max), A0((size_t)nl_max * nl_max), Ct((size_t)nl_max * m_max),
      Y((size_t)nl_max * m_max), G((size_t)m_max * m_max), E((size_t)m_max * ne),
      Phi((size_t)nl_max * ne), R((size_t)m_max * ne), Z((size_t)nl_max * ne),
      T1((size_t)m_max * ne);
  cusolverDnParams_t prm;
  CEM_SOLVER(cusolverDnCreateParams(&prm));
  struct HP {
    cusolverDnParams_t p;
    ~HP() { cusolverDnDestroyParams(p); }
  } hp{prm};
  size_t wd_max = 0, wh_max = 0;
  {
    size_t wd = 0, wh = 0;
    CEM_SOLVER(cusolverDnXpotrf_bufferSize(sol, prm, CUBLAS_FILL_MODE_LOWER, nl_max, CUDA_R_64F,
                                           Al.p, nl_max, CUDA_R_64F, &wd, &wh));
    wd_max = std::max(wd_max, wd);
    wh_max = std::max(wh_max, wh);
    CEM_SOLVER(cusolverDnXpotrf_bufferSize(sol, prm, CUBLAS_FILL_MODE_LOWER, m_max, CUDA_R_64F,
                                           G.p, m_max, CUDA_R_64F, &wd, &wh));
    wd_max = std::max(wd_max, wd);
    wh_max = std::max(wh_max, wh);
  }
  Dv<char> work(std::max<size_t>(wd_max, 1));
  std::vector<char> hwork(std::max<size_t>(wh_max, 1));
  std::vector<int> hinfo(2 * nblk, 0);
  Dv<int> dinfo(2 * nblk);
  PE_CUDA_CHECK(cudaMemsetAsync(dinfo.p, 0, 2 * nblk * sizeof(int), st));
  double worst = 0.0;
  std::vector<double> hphi((size_t)nl_max * ne), hres((size_t)m_max * ne);
  for (int b = 0; b < nblk; ++b) {
    const Patch p = patch_of(g, b);
    const int nl = p.n;
    const int nbx = p.jb1x - p.jb0x, nby = p.jb1y - p.jb0y;
    const int m = nbx * nby * ne;
    k_patch_stiffness<<<grid_for((long long)nl * nl, 256), 256, 0, st>>>(g, p, kap.p, Al.p);
    k_constraints<<<dim3((nl + 255) / 256, m), 256, 0, st>>>(g, p, ne, W.p, Ct.p);
    g_launches += 2;
    PE_CUDA_CHECK(cudaGetLastError());
    PE_CUDA_CHECK(cudaMemcpyAsync(A0.p, Al.p, sizeof(double) * nl * nl, cudaMemcpyDeviceToDevice, st));
    CEM_SOLVER(cusolverDnXpotrf(sol, prm, CUBLAS_FILL_MODE_LOWER, nl, CUDA_R_64F, Al.p, nl,
                                CUDA_R_64F, work.p, wd_max, hwork.data(), wh_max, dinfo.p + 2 * b));
    PE_CUDA_CHECK(cudaMemcpyAsync(Y.p, Ct.p, sizeof(double) * nl * m, cudaMemcpyDeviceToDevice, st));
    CEM_SOLVER(cusolverDnXpotrs(sol, prm, CUBLAS_FILL_MODE_LOWER, nl, m, CUDA_R_64F, Al.p, nl,
                                CUDA_R_64F, Y.p, nl, dinfo.p + 2 * b + 1));
    // G = C Y = Ct^T Y  (m x m)
    CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_T, CUBLAS_OP_N, m, m, nl, &one, Ct.p, nl, Y.p, nl, &zero,
                         G.p, m));
    // targets: this block's rows (its position among the patch blocks, ascending)
    const int bx = b % g.nb, by = b / g.nb;
    const int pos = (by - p.jb0y) * nbx + (bx - p.jb0x);
    std::vector<double> he((size_t)m * ne, 0.0);
    for (int k = 0; k < ne; ++k) he[(size_t)k * m + pos * ne + k] = 1.0;
    PE_CUDA_CHECK(cudaMemcpyAsync(E.p, he.data(), he.size() * 8, cudaMemcpyHostToDevice, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(R.p, he.data(), he.size() * 8, cudaMemcpyHostToDevice, st));
    CEM_SOLVER(cusolverDnXpotrf(sol, prm, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, G.p, m, CUDA_R_64F,
                                work.p, wd_max, hwork.data(), wh_max, dinfo.p + 2 * b));
    CEM_SOLVER(cusolverDnXpotrs(sol, prm, CUBLAS_FILL_MODE_LOWER, m, ne, CUDA_R_64F, G.p, m,
                                CUDA_R_64F, E.p, m, dinfo.p + 2 * b + 1));
    // phi = Y mu  (nl x ne); residual C phi - e
    CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_N, CUBLAS_OP_N, nl, ne, m, &one, Y.p, nl, E.p, m, &zero,
                         Phi.p, nl));
    const double mone = -1.0;
    CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_T, CUBLAS_OP_N, m, ne, nl, &one, Ct.p, nl, Phi.p, nl, &mone,
                         R.p, m));
    // Two steps of iterative refinement on the full KKT system [[A, C^T], [C, 0]]
    // [phi; lambda] = [0; E] (lambda = -mu): the Schur complement G = C A^-1 C^T squares the
    // saddle point's conditioning, the refinement brings phi back to the KKT's own accuracy.
    for (int it = 0; it < 2; ++it) {
      // r1 = C^T mu - A phi  -> Z ;  r2 = E - C phi = -R
      CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_N, CUBLAS_OP_N, nl, ne, m, &one, Ct.p, nl, E.p, m, &zero,
                           Z.p, nl));
      CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_N, CUBLAS_OP_N, nl, ne, nl, &mone, A0.p, nl, Phi.p, nl,
                           &one, Z.p, nl));
      // z = A^-1 r1
      CEM_SOLVER(cusolverDnXpotrs(sol, prm, CUBLAS_FILL_MODE_LOWER, nl, ne, CUDA_R_64F, Al.p, nl,
                                  CUDA_R_64F, Z.p, nl, dinfo.p + 2 * b + 1));
      // dlambda = G^-1 (C z - r2) = G^-1 (C z + R)
      PE_CUDA_CHECK(cudaMemcpyAsync(T1.p, R.p, sizeof(double) * m * ne, cudaMemcpyDeviceToDevice, st));
      CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_T, CUBLAS_OP_N, m, ne, nl, &one, Ct.p, nl, Z.p, nl, &one,
                           T1.p, m));
      CEM_SOLVER(cusolverDnXpotrs(sol, prm, CUBLAS_FILL_MODE_LOWER, m, ne, CUDA_R_64F, G.p, m,
                                  CUDA_R_64F, T1.p, m, dinfo.p + 2 * b + 1));
      // phi += z - Y dlambda ;  mu -= dlambda
      CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_N, CUBLAS_OP_N, nl, ne, m, &mone, Y.p, nl, T1.p, m, &one,
                           Z.p, nl));
      CEM_BLAS(cublasDaxpy(bl, nl * ne, &one, Z.p, 1, Phi.p, 1));
      CEM_BLAS(cublasDaxpy(bl, m * ne, &mone, T1.p, 1, E.p, 1));
      // R = C phi - E_t
      PE_CUDA_CHECK(cudaMemcpyAsync(R.p, he.data(), he.size() * 8, cudaMemcpyHostToDevice, st));
      CEM_BLAS(cublasDgemm(bl, CUBLAS_OP_T, CUBLAS_OP_N, m, ne, nl, &one, Ct.p, nl, Phi.p, nl,
                           &mone, R.p, m));
    }
    PE_CUDA_CHECK(cudaMemcpyAsync(hphi.data(), Phi.p, sizeof(double) * nl * ne,
                                  cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(hres.data(), R.p, sizeof(double) * m * ne,
                                  cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int k = 0; k < ne; ++k)
      for (int i = 0; i < nl; ++i) a.values[a.offsets[b] + (long long)k * nl + i] = hphi[(size_t)k * nl + i];
    for (size_t q = 0; q < (size_t)m * ne; ++q) worst = std::max(worst, std::fabs(hres[q]));
  }
  PE_CUDA_CHECK(cudaMemcpyAsync(hinfo.data(), dinfo.p, 2 * nblk * sizeof(int), cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  for (int b = 0; b < nblk; ++b)
    if (hinfo[2 * b] != 0 || hinfo[2 * b + 1] != 0)
      throw Error{PE_ERR_SOLVER, "singular saddle system on block " + std::to_string(b)};
  if (a.worst) *a.worst = worst;
}

}  // namespace pe

extern "C" int pe_cem_basis(int nx, int nb, int layers, int n_eig, const double* kappa,
                            double kt_scale, double* values, long long* offsets,
                            double* eigenvalues, double* worst, void* stream) {
  if (nx < 2 || nb < 1 || nx % nb || layers < 0 || n_eig < 1 || !kappa || !values || !offsets ||
      n_eig > (nx / nb + 1) * (nx / nb + 1)) {
    pe::set_error("pe_cem_basis: need nb | nx, layers >= 0, 1 <= n_eig <= block nodes, buffers");
    return PE_ERR_ARG;
  }
  for (long long c = 0; c < (long long)nx * nx; ++c)
    if (!(kappa[c] > 0)) {
      pe::set_error("pe_cem_basis: kappa must be strictly positive on every cell");
      return PE_ERR_ARG;
    }
  pe::CemArgs a{nx, nb, layers, n_eig, kappa, kt_scale, values, offsets, eigenvalues, worst,
                (cudaStream_t)stream};
  try {
    pe::cem_impl(a);
    return PE_OK;
  } catch (const pe::Error& e) {
    pe::set_error("pe_cem_basis: " + e.msg);
    return e.code;
  } catch (const std::exception& e) {
    pe::set_error(std::string("pe_cem_basis: ") + e.what());
    return PE_ERR_CUDA;
  }
}

extern "C" long long pe_cem_basis_size(int nx, int nb, int layers, int n_eig) {
  if (nx < 2 || nb < 1 || nx % nb || layers < 0 || n_eig < 1) return -1;
  pe::CemGeom g{nx, nb, nx / nb, layers, (nx / nb + 1) * (nx / nb + 1)};
  long long t = 0;
  for (int b = 0; b < nb * nb; ++b) t += (long long)pe::patch_of(g, b).n * n_eig;
  return t;
}
