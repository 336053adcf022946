// Batched dense inversion by recursive blocked LU with partial (row) pivoting.
//
// This is the factor / solve step of the all-at-once fine solver's setup: the reference
// forms one explicit inverse per time mode, inv(d_k M11 + A11) for k = 0 .. J-1
// (allatonce.py:100-110), and the coarse / sequential factors inv(M11/dt + A11),
// inv(M22) (stepping.py:93-118).  libpe keeps explicit inverses too (every sweep applies
// them hundreds of times as DMMA GEMMs), and builds all of a context's inverses in ONE
// batched pass: the complex shifted matrices enter in their real 2x2-block form
// [[Re, -Im], [Im, Re]] (whose inverse is the real block form of the complex inverse,
// which is exactly the operator layout the sweep applies), so one real kernel family
// serves every factorisation of the setup.
//
// Layout: `batch` row-major n x n matrices, batch stride n*n.  Row pivoting on row-major
// storage swaps contiguous rows.  Recursion (Toledo): factor the left half of a column
// range, swap / triangular-solve / Schur-update the right half with the batched DMMA GEMM
// (gemm_f64), factor the right half, swap the left half.  Leaves (<= 32 columns) run in
// `lu_panel_kernel`: one CTA per matrix, the panel in shared memory when it fits.  The
// inverse is X = U^-1 (L^-1 P) by recursive triangular solves whose off-diagonal updates
// are GEMMs with K = half the block.
//
// Deterministic: fixed reduction orders, first-maximum pivot rule (as LAPACK's idamax).

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "pe.h"
#include "pe_internal.h"

namespace pe {

namespace cg = cooperative_groups;

namespace {

constexpr int LEAF = 32;       // leaf panel / triangular block width
constexpr int PANEL_T = 512;   // threads of the panel kernel
constexpr size_t PANEL_SMEM_MAX = 200 * 1024;

// Factor columns [j0, j0+nb) of rows [j0, n) in place (unit-lower L below the diagonal,
// U on and above).  Row swaps are applied to the panel's own columns only; the caller
// applies piv[j0 .. j0+nb) to the other columns.  info[b] = 1-based index of the first
// exactly-zero pivot (0 if none).
template <bool SMEM>
__global__ void __launch_bounds__(PANEL_T) lu_panel_kernel(int n, int j0, int nb, double* A,
                                                           long long sA, int* piv, int* info) {
  extern __shared__ double sm[];
  __shared__ double prow[LEAF];
  __shared__ double red_v[PANEL_T / 32];
  __shared__ int red_i[PANEL_T / 32];
  __shared__ int s_p;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = n - j0;
  double* Ab = A + blockIdx.x * sA + (long long)j0 * n + j0;
  int* pv = piv + (long long)blockIdx.x * n + j0;
  double* P;
  long long ld;
  if (SMEM) {
    P = sm;
    ld = nb + 1;  // odd row stride: one row per thread is bank-conflict free
    for (long long q = tid; q < (long long)rows * nb; q += PANEL_T) {
      const int r = (int)(q / nb), c = (int)(q - (long long)r * nb);
      P[r * ld + c] = Ab[(long long)r * n + c];
    }
    __syncthreads();
  } else {
    P = Ab;
    ld = n;
  }
  for (int jj = 0; jj < nb; ++jj) {
    // pivot: first row of maximal |a(i, jj)|, i >= jj
    double best = -1.0;
    int bi = rows;
    for (int i = jj + tid; i < rows; i += PANEL_T) {
      const double v = fabs(P[i * ld + jj]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[wid] = best;
      red_i[wid] = bi;
    }
    __syncthreads();
    if (wid == 0) {
      best = lane < PANEL_T / 32 ? red_v[lane] : -1.0;
      bi = lane < PANEL_T / 32 ? red_i[lane] : rows;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        // NaN columns compare false everywhere: keep the diagonal so the NaN propagates
        if (bi >= rows) bi = jj;
        s_p = bi;
        pv[jj] = j0 + bi;
        if (!(best > 0.0) && info[blockIdx.x] == 0) info[blockIdx.x] = j0 + jj + 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (tid < nb) {
      const double a = P[jj * ld + tid], b = P[p * ld + tid];
      P[jj * ld + tid] = b;
      P[p * ld + tid] = a;
      prow[tid] = b;
    }
    __syncthreads();
    const double pvt = prow[jj];
    if (pvt != 0.0) {
      for (int i = jj + 1 + tid; i < rows; i += PANEL_T) {
        double* r = P + i * ld;
        const double l = r[jj] / pvt;
        r[jj] = l;
        for (int c = jj + 1; c < nb; ++c) r[c] = fma(-l, prow[c], r[c]);
      }
    }
    __syncthreads();
  }
  if (SMEM) {
    for (long long q = tid; q < (long long)rows * nb; q += PANEL_T) {
      const int r = (int)(q / nb), c = (int)(q - (long long)r * nb);
      Ab[(long long)r * n + c] = P[r * ld + c];
    }
  }
}

// The same panel for tall matrices: a thread-block cluster per matrix, the panel's rows
// split in contiguous ranges over the cluster's CTAs and held in their shared memory.
// Per column: local pivot candidates, one cluster barrier, every CTA reads all candidates
// through distributed shared memory and picks the same winner; the pivot row is pulled
// from its owner by every CTA (and the displaced row jj by the owner), a second cluster
// barrier, then the owners write the swapped rows and every CTA updates its own rows.
__global__ void __launch_bounds__(PANEL_T) lu_panel_cluster_kernel(int n, int j0, int nb, double* A,
                                                                   long long sA, int* piv,
                                                                   int* info) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int b = blockIdx.x / CS;
  extern __shared__ double sm[];
  __shared__ double prow[LEAF], tmp[LEAF];
  __shared__ double cand_v;
  __shared__ int cand_i;
  __shared__ double red_v[PANEL_T / 32];
  __shared__ int red_i[PANEL_T / 32];
  __shared__ int s_p;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = n - j0;
  const int rp = (rows + CS - 1) / CS;  // >= nb: row jj always lives in CTA 0
  const int r_lo = min(rows, rank * rp), r_hi = min(rows, r_lo + rp);
  const int ld = nb + 1;
  double* Ab = A + b * sA + (long long)j0 * n + j0;
  int* pv = piv + (long long)b * n + j0;
  double* P = sm;
  for (long long q = tid; q < (long long)(r_hi - r_lo) * nb; q += PANEL_T) {
    const int r = (int)(q / nb), c = (int)(q - (long long)r * nb);
    P[r * ld + c] = Ab[(long long)(r_lo + r) * n + c];
  }
  __syncthreads();
  for (int jj = 0; jj < nb; ++jj) {
    double best = -1.0;
    int bi = rows;
    for (int i = max(jj, r_lo) + tid; i < r_hi; i += PANEL_T) {
      const double v = fabs(P[(i - r_lo) * ld + jj]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[wid] = best;
      red_i[wid] = bi;
    }
    __syncthreads();
    if (wid == 0) {
      best = lane < PANEL_T / 32 ? red_v[lane] : -1.0;
      bi = lane < PANEL_T / 32 ? red_i[lane] : rows;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        cand_v = best;
        cand_i = bi;
      }
    }
    cl.sync();
    if (tid == 0) {
      best = -1.0;
      bi = rows;
      for (int q = 0; q < CS; ++q) {
        const double ov = *cl.map_shared_rank(&cand_v, q);
        const int oi = *cl.map_shared_rank(&cand_i, q);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (bi >= rows) bi = jj;
      s_p = bi;
      if (rank == 0) {
        pv[jj] = j0 + bi;
        if (!(best > 0.0) && info[b] == 0) info[b] = j0 + jj + 1;
      }
    }
    __syncthreads();
    const int p = s_p, owner = p / rp;
    if (tid < nb) {
      prow[tid] = cl.map_shared_rank(sm, owner)[(p - owner * rp) * ld + tid];
      if (rank == owner) tmp[tid] = cl.map_shared_rank(sm, 0)[jj * ld + tid];
    }
    cl.sync();
    if (tid < nb) {
      if (rank == 0) P[jj * ld + tid] = prow[tid];
      if (rank == owner && p != jj) P[(p - r_lo) * ld + tid] = tmp[tid];
    }
    __syncthreads();
    const double pvt = prow[jj];
    if (pvt != 0.0) {
      for (int i = max(jj + 1, r_lo) + tid; i < r_hi; i += PANEL_T) {
        double* r = P + (i - r_lo) * ld;
        const double l = r[jj] / pvt;
        r[jj] = l;
        for (int c = jj + 1; c < nb; ++c) r[c] = fma(-l, prow[c], r[c]);
      }
    }
    __syncthreads();
  }
  for (long long q = tid; q < (long long)(r_hi - r_lo) * nb; q += PANEL_T) {
    const int r = (int)(q / nb), c = (int)(q - (long long)r * nb);
    Ab[(long long)(r_lo + r) * n + c] = P[r * ld + c];
  }
}

// Apply the row interchanges piv[r0 .. r0+nr) (in order) to columns [c0, c1) of X.
__global__ void lu_laswp_kernel(int n, int r0, int nr, int c0, int c1, double* X, long long ldx,
                                long long sX, const int* piv) {
  extern __shared__ int sp[];
  const int* pv = piv + (long long)blockIdx.y * n + r0;
  for (int q = threadIdx.x; q < nr; q += blockDim.x) sp[q] = pv[q];
  __syncthreads();
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double* Xb = X + blockIdx.y * sX + c;
  for (int q = 0; q < nr; ++q) {
    const int p = sp[q], r = r0 + q;
    if (p != r) {
      const double a = Xb[(long long)r * ldx], b = Xb[(long long)p * ldx];
      Xb[(long long)r * ldx] = b;
      Xb[(long long)p * ldx] = a;
    }
  }
}

// X = P I: row i of the permuted identity is e_{perm[i]}, perm = the interchanges applied
// to (0, 1, .., n-1).
__global__ void lu_perm_identity_kernel(int n, const int* piv, double* X, long long sX) {
  extern __shared__ int perm[];
  const int* pv = piv + (long long)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < n; ++r) {
      const int p = pv[r];
      if (p != r) {
        const int t = perm[r];
        perm[r] = perm[p];
        perm[p] = t;
      }
    }
  __syncthreads();
  double* Xb = X + blockIdx.x * sX;
  // blockIdx.y owns a contiguous range of rows
  const int per = (n + gridDim.y - 1) / gridDim.y;
  const int i0 = blockIdx.y * per, i1 = min(n, i0 + per);
  for (long long q = (long long)i0 * n + threadIdx.x; q < (long long)i1 * n; q += blockDim.x) {
    const int i = (int)(q / n), j = (int)(q - (long long)i * n);
    Xb[q] = perm[i] == j ? 1.0 : 0.0;
  }
}

// Leaf triangular solves: rows [r0, r0+w) (w <= 32) of X, columns [c0, c1), against the
// diagonal block of the LU factors; one thread per column, the block's rows in registers.
template <bool UPPER>
__global__ void __launch_bounds__(128) lu_trsm_leaf_kernel(int n, int r0, int w, const double* A,
                                                           long long sA, double* X, long long ldx,
                                                           long long sX, int c0, int c1) {
  __shared__ double T[LEAF][LEAF + 1];
  const double* Ab = A + blockIdx.y * sA + (long long)r0 * n + r0;
  for (int q = threadIdx.x; q < w * w; q += blockDim.x) T[q / w][q % w] = Ab[(long long)(q / w) * n + q % w];
  __syncthreads();
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double* Xb = X + blockIdx.y * sX + (long long)r0 * ldx + c;
  double x[LEAF];
#pragma unroll
  for (int r = 0; r < LEAF; ++r) x[r] = r < w ? Xb[(long long)r * ldx] : 0.0;
  if (!UPPER) {
#pragma unroll
    for (int r = 1; r < LEAF; ++r) {
      if (r < w) {
        double s = x[r];
#pragma unroll
        for (int q = 0; q < r; ++q) s = fma(-T[r][q], x[q], s);
        x[r] = s;
      }
    }
  } else {
#pragma unroll
    for (int r = LEAF - 1; r >= 0; --r) {
      if (r < w) {
        double s = x[r];
#pragma unroll
        for (int q = LEAF - 1; q > r; --q)
          if (q < w) s = fma(-T[r][q], x[q], s);
        x[r] = s / T[r][r];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < LEAF; ++r)
    if (r < w) Xb[(long long)r * ldx] = x[r];
}

// In-place transpose of `batch` square row-major matrices: 32 x 32 tile pairs.
__global__ void lu_transpose_inplace_kernel(int n, double* X, long long sX) {
  __shared__ double ta[32][33], tb[32][33];
  const int bx = blockIdx.x, by = blockIdx.y;
  if (bx < by) return;
  double* Xb = X + blockIdx.z * sX;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int i = by * 32 + r, j = bx * 32 + tx;
    if (i < n && j < n) ta[r][tx] = Xb[(long long)i * n + j];
    const int i2 = bx * 32 + r, j2 = by * 32 + tx;
    if (i2 < n && j2 < n) tb[r][tx] = Xb[(long long)i2 * n + j2];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = by * 32 + r, j = bx * 32 + tx;
    if (i < n && j < n) Xb[(long long)i * n + j] = tb[tx][r];
    const int i2 = bx * 32 + r, j2 = by * 32 + tx;
    if (bx != by && i2 < n && j2 < n) Xb[(long long)i2 * n + j2] = ta[tx][r];
  }
}

struct Lu {
  int n, batch;
  double* A;
  long long sA;
  int* piv;
  int* info;
  cudaStream_t st;
  int max_cluster;  // largest cluster size of the tall-panel kernel (0: none)

  static int split(int w) {
    int w1 = ((w / 2 + LEAF - 1) / LEAF) * LEAF;
    if (w1 >= w) w1 = LEAF;
    return w1;
  }

  // C[b] (M x N at row r, column c of X) -= L/U block (rows ar, columns ak, K wide) * X rows
  void gemm_sub(double* X, long long ldx, long long sX, int cr, int cc, int M, int N, int ar,
                int ak, int K, int br) const {
    if (M <= 0 || N <= 0 || K <= 0) return;
    GemmParams p;
    p.M = M;
    p.N = N;
    p.nb1 = batch;
    p.nseg = 1;
    p.seg[0].A = Operand{A + (long long)ar * n + ak, n, 1, sA, 0};
    p.seg[0].B = Operand{X + (long long)br * ldx + cc, ldx, 1, sX, 0};
    p.seg[0].K = K;
    p.C = X + (long long)cr * ldx + cc;
    p.c_i = ldx;
    p.c_j = 1;
    p.c_b1 = sX;
    p.alpha = -1.0;
    p.beta = 1.0;
    p.Cin = p.C;
    gemm_f64(p, st);
  }

  void trsm_leaf(bool upper, int r0, int w, double* X, long long ldx, long long sX, int c0,
                 int c1) const {
    if (c1 <= c0) return;
    dim3 grid((c1 - c0 + 127) / 128, batch);
    if (upper)
      lu_trsm_leaf_kernel<true><<<grid, 128, 0, st>>>(n, r0, w, A, sA, X, ldx, sX, c0, c1);
    else
      lu_trsm_leaf_kernel<false><<<grid, 128, 0, st>>>(n, r0, w, A, sA, X, ldx, sX, c0, c1);
    PE_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }

  // X[r0 : r0+w, c0 : c1] <- L^-1 X, L = the unit-lower block of A at (r0, r0)
  void trsm_lower(int r0, int w, double* X, long long ldx, long long sX, int c0, int c1) const {
    if (w <= LEAF) return trsm_leaf(false, r0, w, X, ldx, sX, c0, c1);
    const int w1 = split(w);
    trsm_lower(r0, w1, X, ldx, sX, c0, c1);
    gemm_sub(X, ldx, sX, r0 + w1, c0, w - w1, c1 - c0, r0 + w1, r0, w1, r0);
    trsm_lower(r0 + w1, w - w1, X, ldx, sX, c0, c1);
  }

  // X[r0 : r0+w, c0 : c1] <- U^-1 X, U = the upper block of A at (r0, r0)
  void trsm_upper(int r0, int w, double* X, long long ldx, long long sX, int c0, int c1) const {
    if (w <= LEAF) return trsm_leaf(true, r0, w, X, ldx, sX, c0, c1);
    const int w1 = split(w);
    trsm_upper(r0 + w1, w - w1, X, ldx, sX, c0, c1);
    gemm_sub(X, ldx, sX, r0, c0, w1, c1 - c0, r0, r0 + w1, w - w1, r0 + w1);
    trsm_upper(r0, w1, X, ldx, sX, c0, c1);
  }

  void laswp(int r0, int nr, int c0, int c1, double* X, long long ldx, long long sX) const {
    if (c1 <= c0 || nr <= 0) return;
    dim3 grid((c1 - c0 + 127) / 128, batch);
    lu_laswp_kernel<<<grid, 128, sizeof(int) * nr, st>>>(n, r0, nr, c0, c1, X, ldx, sX, piv);
    PE_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }

  void panel(int j0, int nb) const {
    const int rows = n - j0;
    const size_t need = sizeof(double) * (size_t)rows * (nb + 1);
    ++g_launches;
    if (need <= PANEL_SMEM_MAX) {
      lu_panel_kernel<true><<<batch, PANEL_T, need, st>>>(n, j0, nb, A, sA, piv, info);
      PE_CUDA_CHECK(cudaGetLastError());
      return;
    }
    for (int cs = 2; cs <= max_cluster; cs *= 2) {
      const int rp = (rows + cs - 1) / cs;
      const size_t sm = sizeof(double) * (size_t)rp * (nb + 1);
      if (sm > PANEL_SMEM_MAX) continue;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(batch * cs);
      cfg.blockDim = dim3(PANEL_T);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, lu_panel_cluster_kernel, n, j0, nb, A, sA, piv, info));
      return;
    }
    lu_panel_kernel<false><<<batch, PANEL_T, 0, st>>>(n, j0, nb, A, sA, piv, info);
    PE_CUDA_CHECK(cudaGetLastError());
  }

  // factor columns [j0, j0+w) of rows [j0, n); interchanges applied within those columns
  void factor(int j0, int w) const {
    if (w <= LEAF) return panel(j0, w);
    const int w1 = split(w), w2 = w - w1;
    factor(j0, w1);
    laswp(j0, w1, j0 + w1, j0 + w, A, n, sA);
    trsm_lower(j0, w1, A, n, sA, j0 + w1, j0 + w);
    gemm_sub(A, n, sA, j0 + w1, j0 + w1, n - j0 - w1, w2, j0 + w1, j0, w1, j0);
    factor(j0 + w1, w2);
    laswp(j0 + w1, w2, j0, j0 + w1, A, n, sA);
  }
};

}  // namespace

// PE_LU_CLUSTER caps the tall-panel cluster size (tests: 0 forces the global-memory panel)
static int panel_max_cluster() {
  const char* e = std::getenv("PE_LU_CLUSTER");
  return e ? std::atoi(e) : 16;
}

void batched_lu_inverse(int n, int batch, double* A, double* Ainv, int* piv, int* info,
                        cudaStream_t st) {
  if (n <= 0 || batch <= 0) return;
  if ((size_t)n * sizeof(int) > PANEL_SMEM_MAX)
    throw Error{PE_ERR_ARG, "batched_lu_inverse: n = " + std::to_string(n) + " exceeds " +
                                std::to_string(PANEL_SMEM_MAX / sizeof(int))};
  static bool attr_set = false;
  if (!attr_set) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(lu_panel_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)PANEL_SMEM_MAX));
    PE_CUDA_CHECK(cudaFuncSetAttribute(lu_panel_cluster_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)PANEL_SMEM_MAX));
    PE_CUDA_CHECK(cudaFuncSetAttribute(lu_panel_cluster_kernel,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    PE_CUDA_CHECK(cudaFuncSetAttribute(lu_perm_identity_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)PANEL_SMEM_MAX));
    attr_set = true;
  }
  PE_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int) * (size_t)batch, st));
  const long long sA = (long long)n * n;
  // The factorisation runs on A^T and the result is transposed back: a solve against I
  // gets the COLUMNS of an inverse backward stably (A^T Y = I to round-off), so the rows
  // of Ainv = Y^T satisfy Ainv A = I to round-off, which is the residual that bounds the
  // error of applying Ainv to a vector (|Ainv b - x| <= |Ainv A - I| |x|).  The other
  // order would leave Ainv A - I at cond(A) eps.
  const dim3 tgrid((n + 31) / 32, (n + 31) / 32, batch), tblock(32, 8);
  lu_transpose_inplace_kernel<<<tgrid, tblock, 0, st>>>(n, A, sA);
  PE_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  Lu lu{n, batch, A, sA, piv, info, st, panel_max_cluster()};
  lu.factor(0, n);
  lu_perm_identity_kernel<<<dim3(batch, std::max(1, std::min(64, n / 64))), 1024,
                            sizeof(int) * (size_t)n, st>>>(n, piv, Ainv, sA);
  PE_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  lu.trsm_lower(0, n, Ainv, n, sA, 0, n);
  lu.trsm_upper(0, n, Ainv, n, sA, 0, n);
  lu_transpose_inplace_kernel<<<tgrid, tblock, 0, st>>>(n, Ainv, sA);
  PE_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

namespace {

// block form [[Re, -Im], [Im, Re]] of d_k M + A for modes k = 0 .. J/2 (blockIdx.y)
__global__ void shifted_family_kernel(int n, int J, double dt, double om_r, const double* M,
                                      const double* A, double* S) {
  const int k = blockIdx.y;
  double sn, cs;
  sincospi(-2.0 * (double)k / (double)J, &sn, &cs);
  const double dre = (1.0 - om_r * cs) / dt, dim = (-om_r * sn) / dt;
  const long long n2 = 2LL * n;
  double* Sk = S + (long long)k * n2 * n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t % n;
    const double re = dre * M[t] + A[t], im = dim * M[t];
    Sk[i * n2 + j] = re;
    Sk[i * n2 + n + j] = -im;
    Sk[(i + n) * n2 + j] = im;
    Sk[(i + n) * n2 + n + j] = re;
  }
}

// planar (J, n, n) outputs from the block-form inverses; modes above J/2 by conjugation
__global__ void unpack_family_kernel(int n, int J, const double* X, double* inv_re,
                                     double* inv_im) {
  const int k = blockIdx.y;  // 0 .. J-1
  const int src = k <= J / 2 ? k : J - k;
  const double sg = k <= J / 2 ? 1.0 : -1.0;
  const long long n2 = 2LL * n;
  const double* Xk = X + (long long)src * n2 * n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t % n;
    inv_re[(long long)k * n * n + t] = Xk[i * n2 + j];
    inv_im[(long long)k * n * n + t] = sg * Xk[(i + n) * n2 + j];
  }
}

struct Scratch {
  void* p = nullptr;
  explicit Scratch(size_t bytes) {
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw Error{PE_ERR_NOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed"};
    }
  }
  ~Scratch() { cudaFree(p); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

}  // namespace

void shifted_inverses(int d1, int J, double dt, double alpha, const double* M11,
                      const double* A11, double* inv_re, double* inv_im, cudaStream_t st) {
  if (d1 <= 0 || J <= 0) return;
  const int nm = J / 2 + 1, n2 = 2 * d1;
  const size_t per = (size_t)n2 * n2;
  Scratch S(sizeof(double) * nm * per), X(sizeof(double) * nm * per),
      piv(sizeof(int) * (size_t)nm * n2), info(sizeof(int) * (size_t)nm);
  const int gx = (int)std::min<long long>(1024, ((long long)d1 * d1 + 255) / 256);
  shifted_family_kernel<<<dim3(gx, nm), 256, 0, st>>>(d1, J, dt, std::pow(alpha, 1.0 / J), M11,
                                                       A11, (double*)S.p);
  PE_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  batched_lu_inverse(n2, nm, (double*)S.p, (double*)X.p, (int*)piv.p, (int*)info.p, st);
  unpack_family_kernel<<<dim3(gx, J), 256, 0, st>>>(d1, J, (const double*)X.p, inv_re, inv_im);
  PE_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  std::vector<int> h((size_t)nm);
  PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), info.p, sizeof(int) * nm, cudaMemcpyDeviceToHost, st));
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  for (int k = 0; k < nm; ++k)
    if (h[k] != 0)
      throw Error{PE_ERR_SOLVER, "singular shifted matrix d_k M11 + A11 (mode " +
                                     std::to_string(k) + ", zero pivot " + std::to_string(h[k]) +
                                     ")"};
}

}  // namespace pe
