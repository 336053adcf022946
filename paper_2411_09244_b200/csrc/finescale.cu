// Fine-scale accuracy path: the fine backward-Euler reference solve
// (fem.py:292-318 reference_solve) and the Eq (31) relative-error series of the parareal
// iterates (experiment.py:320-325 relative_error, :348-354 the per-iteration series;
// msbasis.py:448-450 reconstruct; fem.py:272-274 norm).
//
// Reference solve.  The fine operator K = M/dt + A is constant, so the setup factorises it
// once (cuSOLVER 64-bit potrf + potrs against I: explicit SPD inverse) and folds the mass term in:
//     u_{s+1} = R u_s + c,   R = K^-1 M / dt (dense, row-major),  c = K^-1 b.
// Every time step is then ONE HBM-streaming GEMV over R (n^2 * 8 bytes), instead of the
// reference's two sparse triangular sweeps (splu.solve), which run one row at a time.
// The step chain is sequential in time; each step is a grid-wide dependency, so it is one
// launch per step on the caller's stream.
//
// Error series.  Fine reconstructions Y_k = [Psi1 Psi2] x_k for all K iterates at once
// (CSR SpMM, one warp per fine row), D_k = ref - Y_k, then ||D_k||_M = sqrt(D_k^T M D_k)
// with a deterministic two-level reduction (fixed-order block partials, then a fixed-order
// sum per column).  Row K of D is ref itself, which gives the denominator ||ref||_M.

#include <cusolverDn.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "pe.h"
#include "finescale.h"
#include "mbar.cuh"
#include "pe_internal.h"

namespace pe {

extern long long g_launches;

namespace {

#define FS_SOLVER_CHECK(x)                                                              \
  do {                                                                                  \
    cusolverStatus_t _s = (x);                                                          \
    if (_s != CUSOLVER_STATUS_SUCCESS)                                                  \
      throw Error{PE_ERR_SOLVER, std::string(#x) + " failed: " + std::to_string(_s)};   \
  } while (0)

template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) {
    if (n) {
      cudaError_t e = cudaMalloc(&p, n * sizeof(T));
      if (e != cudaSuccess)
        throw Error{PE_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(n * sizeof(T)) +
                                      " B): " + cudaGetErrorString(e)};
    }
  }
  ~Dev() { cudaFree(p); }
  void reset() {
    cudaFree(p);  // synchronises the device first
    p = nullptr;
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

struct Csr {
  int n = 0, nnz = 0;
  Dev<int> ptr, idx;
  Dev<double> val;
  Csr(int rows, const int* hptr, const int* hidx, const double* hval)
      : n(rows), nnz(hptr[rows]), ptr(rows + 1), idx(hptr[rows]), val(hptr[rows]) {
    PE_CUDA_CHECK(cudaMemcpy(ptr.p, hptr, (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (nnz) {
      PE_CUDA_CHECK(cudaMemcpy(idx.p, hidx, nnz * sizeof(int), cudaMemcpyHostToDevice));
      PE_CUDA_CHECK(cudaMemcpy(val.p, hval, nnz * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
};

// K(i, j) = M(i, j) / dt + A(i, j), dense column-major with leading dimension ld (K is
// symmetric, so the storage order only matters for the padding).  One thread per row.
__global__ void k_scatter_K(int n, long long ld, const int* mp, const int* mi, const double* mv,
                            const int* ap, const int* ai, const double* av, double inv_dt,
                            double* K) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int t = mp[i]; t < mp[i + 1]; ++t) K[(long long)mi[t] * ld + i] += mv[t] * inv_dt;
  for (int t = ap[i]; t < ap[i + 1]; ++t) K[(long long)ai[t] * ld + i] += av[t];
}

// B = I (column-major, leading dimension ld): the right-hand sides of K X = I.
__global__ void k_identity(int n, long long ld, double* B) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long j = t / n, i = t % n;
  if (j >= n) return;
  B[j * ld + i] = (i == j) ? 1.0 : 0.0;
}

// R(i, :) = Kinv(i, :) M / dt  (row-major R, ld).  Kinv symmetric: Kinv(i, l) is read
// from column i of the column-major buffer, i.e. contiguous in l.  M symmetric: column j
// of M equals row j.  One warp per (i, 32-column chunk) keeps Kinv(i, :) in L1/L2.
__global__ void k_form_R(int n, long long ld, const double* __restrict__ Kinv,
                         const int* __restrict__ mp, const int* __restrict__ mi,
                         const double* __restrict__ mv, double inv_dt, double* __restrict__ R) {
  int i = blockIdx.y;
  const double* ki = Kinv + (long long)i * ld;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = mp[j]; t < mp[j + 1]; ++t) s = fma(ki[mi[t]], mv[t], s);
    R[(long long)i * ld + j] = s * inv_dt;
  }
}

// y = A x (+ c), A row-major n x n with leading dimension ld (multiple of 2), one warp
// per row, 16-byte loads, four in flight per lane, fixed-order shuffle reduction.
__global__ void __launch_bounds__(256) k_gemv_rows(int n, long long ld,
                                                   const double* __restrict__ A,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ c,
                                                   double* __restrict__ y) {
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double2* a2 = reinterpret_cast<const double2*>(A + (long long)row * ld);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  int n2 = n >> 1;
  double s0 = 0.0, s1 = 0.0;
  int t = lane;
  for (; t + 96 < n2; t += 128) {
    double2 a0 = __ldcs(a2 + t), a1 = __ldcs(a2 + t + 32), a2v = __ldcs(a2 + t + 64),
            a3 = __ldcs(a2 + t + 96);
    double2 b0 = __ldg(x2 + t), b1 = __ldg(x2 + t + 32), b2 = __ldg(x2 + t + 64),
            b3 = __ldg(x2 + t + 96);
    s0 = fma(a0.x, b0.x, s0); s1 = fma(a0.y, b0.y, s1);
    s0 = fma(a1.x, b1.x, s0); s1 = fma(a1.y, b1.y, s1);
    s0 = fma(a2v.x, b2.x, s0); s1 = fma(a2v.y, b2.y, s1);
    s0 = fma(a3.x, b3.x, s0); s1 = fma(a3.y, b3.y, s1);
  }
  for (; t < n2; t += 32) {
    double2 a0 = __ldcs(a2 + t), b0 = __ldg(x2 + t);
    s0 = fma(a0.x, b0.x, s0); s1 = fma(a0.y, b0.y, s1);
  }
  if ((n & 1) && lane == 0) s0 = fma(A[(long long)row * ld + n - 1], x[n - 1], s0);
  double s = s0 + s1;
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = c ? s + c[row] : s;
}

// D(k, i) = ref(i) - sum_j P(i, j) X(k, j) for k < K, D(K, i) = ref(i).  P: CSR n x d.
// One warp per fine row i; lanes split the row's nonzeros, fixed-order shuffle sum.
__global__ void k_reconstruct_diff(int n, int d, int K, const int* __restrict__ pp,
                                   const int* __restrict__ pi, const double* __restrict__ pv,
                                   const double* __restrict__ X, const double* __restrict__ ref,
                                   double* __restrict__ D) {
  int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (i >= n) return;
  int b = pp[i], e = pp[i + 1];
  for (int k = 0; k < K; ++k) {
    const double* xk = X + (long long)k * d;
    double s = 0.0;
    for (int t = b + lane; t < e; t += 32) s = fma(pv[t], xk[pi[t]], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) D[(long long)k * n + i] = ref[i] - s;
  }
  if (lane == 0) D[(long long)K * n + i] = ref[i];
}

// partial[k * nblk + blk] = sum over this block's rows i of D(k,i) * (M D(k,:))(i).
__global__ void __launch_bounds__(256) k_mnorm_partial(int n, const int* __restrict__ mp,
                                                       const int* __restrict__ mi,
                                                       const double* __restrict__ mv,
                                                       const double* __restrict__ D,
                                                       double* __restrict__ partial) {
  __shared__ double red[256];
  int k = blockIdx.y;
  const double* dk = D + (long long)k * n;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = mp[i]; t < mp[i + 1]; ++t) s = fma(mv[t], dk[mi[t]], s);
    acc = fma(dk[i], s, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(long long)k * gridDim.x + blockIdx.x] = red[0];
}

__global__ void k_mnorm_final(int nblk, int K1, const double* __restrict__ partial,
                              double* __restrict__ norms) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K1) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(long long)k * nblk + b];
  norms[k] = sqrt(s);
}

// ---- packed symmetric path (n >= kSymMin): K^-1 is symmetric, so each step streams only
// its lower-triangle tiles (half the bytes of R).  Tile (I, J), J <= I, of B x B doubles is
// stored row-major at tile index I (I + 1) / 2 + J (zero padded past n).  One CTA per tile
// produces the tile's row sums T v_J (rowpart) and, off the diagonal, its column sums
// T^T v_I (colpart, the mirrored upper tile); k_sym_reduce adds them per row in a fixed
// order.  Per step: v = M u / dt + b (k_rhs), the tile pass, the reduction.
constexpr int kB = 128;
constexpr int kSymMin = 4096;

__device__ __forceinline__ int tri_row(int t) {
  int I = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(I + 1) * (I + 2) / 2 <= t) ++I;
  while ((long long)I * (I + 1) / 2 > t) --I;
  return I;
}

__global__ void k_pack_tiles(int n, long long ld, const double* __restrict__ Kinv,
                             double* __restrict__ T) {
  int t = blockIdx.x;
  int I = tri_row(t), J = t - I * (I + 1) / 2;
  double* dst = T + (size_t)t * kB * kB;
  for (int idx = threadIdx.x; idx < kB * kB; idx += blockDim.x) {
    int r = idx / kB, c = idx % kB;
    long long gi = (long long)I * kB + r, gj = (long long)J * kB + c;
    dst[idx] = (gi < n && gj < n) ? Kinv[gi * ld + gj] : 0.0;
  }
}

// v(i) = (M u)(i) / dt + b(i), i < n (rows past n stay zero)
__global__ void k_rhs(int n, const int* __restrict__ mp, const int* __restrict__ mi,
                      const double* __restrict__ mv, double inv_dt, const double* __restrict__ u,
                      const double* __restrict__ b, double* __restrict__ v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int t = mp[i]; t < mp[i + 1]; ++t) s = fma(mv[t], u[mi[t]], s);
  v[i] = fma(s, inv_dt, b[i]);
}

__global__ void __launch_bounds__(256) k_sym_tiles(const double* __restrict__ T,
                                                   const double* __restrict__ v,
                                                   double* __restrict__ rowpart,
                                                   double* __restrict__ colpart) {
  __shared__ double rowred[2][kB];
  __shared__ double colred[4][kB];
  const int t = blockIdx.x;
  const int I = tri_row(t), J = t - I * (I + 1) / 2;
  const int cp = threadIdx.x & 63, rg = threadIdx.x >> 6, lane = threadIdx.x & 31;
  const double2* tile = reinterpret_cast<const double2*>(T + (size_t)t * kB * kB);
  const double2 vJ = reinterpret_cast<const double2*>(v + (size_t)J * kB)[cp];
  const double* vI = v + (size_t)I * kB + rg * 32;
  double rp[32];
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    double2 a = __ldcs(tile + (rg * 32 + r) * (kB / 2) + cp);
    double vi = __ldg(vI + r);
    c0 = fma(a.x, vi, c0);
    c1 = fma(a.y, vi, c1);
    rp[r] = fma(a.x, vJ.x, a.y * vJ.y);
  }
  // transpose-reduce the 32 row partials across the warp: lane L ends with row L's sum
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      double send = up ? rp[i] : rp[i + s];
      double keep = up ? rp[i + s] : rp[i];
      rp[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  rowred[(threadIdx.x >> 5) & 1][rg * 32 + lane] = rp[0];
  colred[rg][2 * cp] = c0;
  colred[rg][2 * cp + 1] = c1;
  __syncthreads();
  if (threadIdx.x < kB) {
    rowpart[(size_t)t * kB + threadIdx.x] = rowred[0][threadIdx.x] + rowred[1][threadIdx.x];
  } else if (I != J) {
    int c = threadIdx.x - kB;
    colpart[(size_t)t * kB + c] = ((colred[0][c] + colred[1][c]) + colred[2][c]) + colred[3][c];
  }
}


// Persistent TMA-bulk variant of k_sym_tiles: one CTA per SM walks tiles t = blockIdx.x,
// + gridDim.x, ...; each tile is two 64 KB half-tiles (64 rows), streamed global -> shared
// by cp.async.bulk into a 3-stage ring (mbarrier complete_tx), so the next half-tiles are
// in flight while the CTA reduces the current one.  Same sums as k_sym_tiles, fixed order.
constexpr int kHalfRows = 64;
constexpr int kStages = 3;
constexpr unsigned kHalfBytes = kHalfRows * kB * sizeof(double);

__global__ void __launch_bounds__(256, 1) k_sym_tiles_tma(const double* __restrict__ T,
                                                          const double* __restrict__ v,
                                                          int ntiles,
                                                          double* __restrict__ rowpart,
                                                          double* __restrict__ colpart) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // kStages x (64 x 64) double2
  __shared__ __align__(8) unsigned long long full[kStages];
  __shared__ double rowred[2][2][kHalfRows];
  __shared__ double colred[4][kB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cp = tid & 63, rg = tid >> 6;  // column pair, 16-row group
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int units = 2 * my_tiles;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int u) {
    int t = blockIdx.x + (u >> 1) * gridDim.x;
    const double* src = T + (size_t)t * kB * kB + (size_t)(u & 1) * kHalfRows * kB;
    unsigned bar = smem_u32(&full[u % kStages]);
    mbar_expect_tx(bar, kHalfBytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(buf + (size_t)(u % kStages) * kHalfRows * (kB / 2))), "l"(src),
        "r"(kHalfBytes), "r"(bar)
        : "memory");
  };
  if (tid == 0)
    for (int u = 0; u < kStages && u < units; ++u) issue(u);
  double c0 = 0.0, c1 = 0.0;
  for (int u = 0; u < units; ++u) {
    const int t = blockIdx.x + (u >> 1) * gridDim.x, h = u & 1;
    const int I = tri_row(t), J = t - I * (I + 1) / 2;
    mbar_wait_cta(smem_u32(&full[u % kStages]), (u / kStages) & 1);
    const double2* tile = buf + (size_t)(u % kStages) * kHalfRows * (kB / 2);
    const double2 vJ = reinterpret_cast<const double2*>(v + (size_t)J * kB)[cp];
    const double* vI = v + (size_t)I * kB + h * kHalfRows + rg * 16;
    if (h == 0) c0 = c1 = 0.0;
    double rp[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double2 a = tile[(rg * 16 + r) * (kB / 2) + cp];
      double vi = __ldg(vI + r);
      c0 = fma(a.x, vi, c0);
      c1 = fma(a.y, vi, c1);
      rp[r] = fma(a.x, vJ.x, a.y * vJ.y);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) rp[i] += __shfl_xor_sync(0xffffffffu, rp[i], 16);
#pragma unroll
    for (int s2 = 8; s2 >= 1; s2 >>= 1) {
      const bool up = lane & s2;
#pragma unroll
      for (int i = 0; i < s2; ++i) {
        double send = up ? rp[i] : rp[i + s2];
        double keep = up ? rp[i + s2] : rp[i];
        rp[i] = keep + __shfl_xor_sync(0xffffffffu, send, s2);
      }
    }
    if (lane < 16) rowred[u & 1][w & 1][rg * 16 + lane] = rp[0];
    if (h == 1) {
      colred[rg][2 * cp] = c0;
      colred[rg][2 * cp + 1] = c1;
    }
    __syncthreads();  // stage u % kStages fully read; rowred / colred complete
    if (tid == 0 && u + kStages < units) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(u + kStages);
    }
    if (tid < kHalfRows) {
      rowpart[(size_t)t * kB + h * kHalfRows + tid] = rowred[u & 1][0][tid] + rowred[u & 1][1][tid];
    } else if (h == 1 && tid >= kB && I != J) {
      int c = tid - kB;
      colpart[(size_t)t * kB + c] = ((colred[0][c] + colred[1][c]) + colred[2][c]) + colred[3][c];
    }
  }
}

// y(i) for the 64 rows of half a band K: 16 slices per row each sum a fixed strided subset
// of the band's nb partial vectors (rowparts J <= K, then colparts I > K), coalesced over
// rows; the slices are combined in a fixed order through shared memory.
constexpr int kRedRows = 64, kRedSlices = 16;
__global__ void __launch_bounds__(kRedRows * kRedSlices) k_sym_reduce(
    int n, int nb, const double* __restrict__ rowpart, const double* __restrict__ colpart,
    double* __restrict__ y) {
  __shared__ double red[kRedSlices][kRedRows];
  const int K = blockIdx.x >> 1;
  const int r = (blockIdx.x & 1) * kRedRows + (threadIdx.x % kRedRows);
  const int sl = threadIdx.x / kRedRows;
  const size_t base = (size_t)K * (K + 1) / 2;
  double s = 0.0;
  for (int j = sl; j < nb; j += kRedSlices) {
    const double* src = j <= K ? rowpart + (base + j) * kB
                               : colpart + ((size_t)j * (j + 1) / 2 + K) * kB;
    s += src[r];
  }
  red[sl][threadIdx.x % kRedRows] = s;
  __syncthreads();
  if (sl == 0) {
    double t = red[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < kRedSlices; ++q) t += red[q][threadIdx.x];
    int i = K * kB + r;
    if (i < n) y[i] = t;
  }
}

long long padded_ld(int n) { return ((long long)n + 3) & ~3LL; }

}  // namespace

static int fs_guard(const char* what, void (*fn)(void*), void* arg) {
  try {
    fn(arg);
    return PE_OK;
  } catch (const Error& e) {
    set_error(std::string(what) + ": " + e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(std::string(what) + ": " + e.what());
    return PE_ERR_CUDA;
  }
}

void fine_rhs(int n, const int* mp, const int* mi, const double* mv, double inv_dt,
              const double* u, const double* b, double* v, cudaStream_t st) {
  k_rhs<<<(n + 255) / 256, 256, 0, st>>>(n, mp, mi, mv, inv_dt, u, b, v);
}

static void ref_solve_impl(void* vp) {
  RefSolveArgs& a = *static_cast<RefSolveArgs*>(vp);
  const int n = a.n;
  // large banded operators: the block-tridiagonal chain solver (finechain.cu)
  if (fine_chain_applicable(n, a.mp, a.mi, a.ap, a.ai)) return fine_chain_solve(a);
  if (n > 65535)
    throw Error{PE_ERR_ARG, "fine problems above 65535 interior nodes need a banded operator "
                            "(half-bandwidth <= 512) for the chain solver"};
  const double dt = a.t_end / a.n_steps;
  const double inv_dt = 1.0 / dt;
  const long long ld = padded_ld(n);
  Csr M(n, a.mp, a.mi, a.mv), A(n, a.ap, a.ai, a.av);
  Dev<double> K((size_t)ld * n), R((size_t)ld * n), bc(2 * (size_t)n);
  Dev<int> info(1);
  PE_CUDA_CHECK(cudaMemsetAsync(K.p, 0, sizeof(double) * ld * n, a.st));
  PE_CUDA_CHECK(cudaMemcpyAsync(bc.p, a.b, n * sizeof(double), cudaMemcpyHostToDevice, a.st));
  k_scatter_K<<<(n + 255) / 256, 256, 0, a.st>>>(n, ld, M.ptr.p, M.idx.p, M.val.p, A.ptr.p,
                                                 A.idx.p, A.val.p, inv_dt, K.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());

  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  FS_SOLVER_CHECK(cusolverDnCreate(&h));
  struct HGuard {
    cusolverDnHandle_t h;
    cusolverDnParams_t* p;
    ~HGuard() {
      if (*p) cusolverDnDestroyParams(*p);
      cusolverDnDestroy(h);
    }
  } hg{h, &prm};
  FS_SOLVER_CHECK(cusolverDnCreateParams(&prm));
  FS_SOLVER_CHECK(cusolverDnSetStream(h, a.st));
  // 64-bit API: n * ld exceeds 2^31 at the larger fine grids
  size_t wd = 0, wh = 0;
  FS_SOLVER_CHECK(cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, K.p,
                                              ld, CUDA_R_64F, &wd, &wh));
  {
    Dev<char> work(wd + 16);
    std::vector<char> hwork(wh + 16);
    FS_SOLVER_CHECK(cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, K.p, ld,
                                     CUDA_R_64F, work.p, wd, hwork.data(), wh, info.p));
    int hinfo = 0;
    PE_CUDA_CHECK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, a.st));
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
    if (hinfo != 0)
      throw Error{PE_ERR_SOLVER, "M/dt + A is not positive definite (potrf info " +
                                     std::to_string(hinfo) + ")"};
  }
  // Kinv = K^-1 I (two triangular solves against the identity; symmetric, full storage)
  long long tot = (long long)n * n;
  k_identity<<<(unsigned)((tot + 255) / 256), 256, 0, a.st>>>(n, ld, R.p);
  ++g_launches;
  FS_SOLVER_CHECK(cusolverDnXpotrs(h, prm, CUBLAS_FILL_MODE_LOWER, n, n, CUDA_R_64F, K.p, ld,
                                   CUDA_R_64F, R.p, ld, info.p));
  {
    int hinfo = 0;
    PE_CUDA_CHECK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, a.st));
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
    if (hinfo != 0)
      throw Error{PE_ERR_SOLVER, "potrs against the identity failed (info " +
                                     std::to_string(hinfo) + ")"};
  }
  // c = Kinv b; then R = Kinv M / dt, written over the factor's buffer
  k_gemv_rows<<<(n + 7) / 8, 256, 0, a.st>>>(n, ld, R.p, bc.p, nullptr, bc.p + n);
  ++g_launches;
  const bool sym = n >= kSymMin && !getenv("PE_FINE_NO_SYM");
  if (sym) {  // the factor is dead once K^-1 and c exist
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
    K.reset();
  }
  const int nbk = (n + kB - 1) / kB;
  const size_t ntiles = sym ? (size_t)nbk * (nbk + 1) / 2 : 0;
  Dev<double> T(ntiles * kB * kB), rowpart(ntiles * kB), colpart(ntiles * kB),
      vpad(sym ? (size_t)nbk * kB : 0);
  double* Rm = K.p;
  const bool tma = sym && !getenv("PE_FINE_NO_TMA");
  int tma_grid = 0;
  if (tma) {
    int dev = 0, nsm = 0;
    PE_CUDA_CHECK(cudaGetDevice(&dev));
    PE_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    tma_grid = (int)std::min<size_t>((size_t)nsm, ntiles);
    PE_CUDA_CHECK(cudaFuncSetAttribute(k_sym_tiles_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kStages * kHalfBytes)));
  }
  if (sym) {
    k_pack_tiles<<<(unsigned)ntiles, 256, 0, a.st>>>(n, ld, R.p, T.p);
    ++g_launches;
    PE_CUDA_CHECK(cudaMemsetAsync(vpad.p, 0, sizeof(double) * nbk * kB, a.st));
    PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
    R.reset();  // the steps read only the packed tiles (n^2 / 2)
  } else {
    dim3 gR((n + 255) / 256 < 8 ? (n + 255) / 256 : 8, n);
    k_form_R<<<gR, 256, 0, a.st>>>(n, ld, R.p, M.ptr.p, M.idx.p, M.val.p, inv_dt, K.p);
    ++g_launches;
  }
  PE_CUDA_CHECK(cudaGetLastError());
  PE_CUDA_CHECK(cudaStreamSynchronize(a.st));

  const size_t nb = (size_t)n * sizeof(double);
  size_t traj_rows = a.keep ? (size_t)a.n_steps + 1 : 3;  // else [u0, ping, pong]
  Dev<double> U(traj_rows * ld);  // rows at 32-byte aligned stride ld (16-byte GEMV loads)
  if (a.u0)
    PE_CUDA_CHECK(cudaMemcpyAsync(U.p, a.u0, nb, cudaMemcpyHostToDevice, a.st));
  else
    PE_CUDA_CHECK(cudaMemsetAsync(U.p, 0, nb, a.st));
  struct EventPair {  // destroyed on every exit path, including a thrown CUDA error
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~EventPair() {
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    }
  } ev;
  cudaEvent_t& e0 = ev.e0;
  cudaEvent_t& e1 = ev.e1;
  if (a.step_ms) {
    PE_CUDA_CHECK(cudaEventCreate(&e0));
    PE_CUDA_CHECK(cudaEventCreate(&e1));
    PE_CUDA_CHECK(cudaEventRecord(e0, a.st));
  }
  for (int s = 0; s < a.n_steps; ++s) {
    const double* src = U.p + (size_t)(a.keep || s == 0 ? s : 1 + ((s - 1) & 1)) * ld;
    double* dst = U.p + (size_t)(a.keep ? s + 1 : 1 + (s & 1)) * ld;
    if (sym) {
      k_rhs<<<(n + 255) / 256, 256, 0, a.st>>>(n, M.ptr.p, M.idx.p, M.val.p, inv_dt, src, bc.p,
                                               vpad.p);
      if (tma)
        k_sym_tiles_tma<<<tma_grid, 256, kStages * kHalfBytes, a.st>>>(T.p, vpad.p, (int)ntiles,
                                                                     rowpart.p, colpart.p);
      else
        k_sym_tiles<<<(unsigned)ntiles, 256, 0, a.st>>>(T.p, vpad.p, rowpart.p, colpart.p);
      k_sym_reduce<<<2 * nbk, kRedRows * kRedSlices, 0, a.st>>>(n, nbk, rowpart.p, colpart.p, dst);
      g_launches += 3;
    } else {
      k_gemv_rows<<<(n + 7) / 8, 256, 0, a.st>>>(n, ld, Rm, src, bc.p + n, dst);
      ++g_launches;
    }
  }
  PE_CUDA_CHECK(cudaGetLastError());
  if (a.step_ms) {
    PE_CUDA_CHECK(cudaEventRecord(e1, a.st));
    PE_CUDA_CHECK(cudaEventSynchronize(e1));
    PE_CUDA_CHECK(cudaEventElapsedTime(a.step_ms, e0, e1));
  }
  if (a.keep) {
    PE_CUDA_CHECK(cudaMemcpy2DAsync(a.states_h, nb, U.p, ld * sizeof(double), nb, traj_rows,
                                    cudaMemcpyDeviceToHost, a.st));
  } else {
    PE_CUDA_CHECK(cudaMemcpyAsync(a.states_h, U.p, nb, cudaMemcpyDeviceToHost, a.st));
    PE_CUDA_CHECK(cudaMemcpyAsync(a.states_h + n, U.p + (size_t)(1 + ((a.n_steps - 1) & 1)) * ld, nb,
                                  cudaMemcpyDeviceToHost, a.st));
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
}

struct ErrArgs {
  int n, d, K;
  const int *pp, *pi, *mp, *mi;
  const double *pv, *mv, *ref, *X;
  double* norms_h;
  cudaStream_t st;
};

static void err_impl(void* vp) {
  ErrArgs& a = *static_cast<ErrArgs*>(vp);
  const int n = a.n, K1 = a.K + 1;
  Csr P(n, a.pp, a.pi, a.pv), M(n, a.mp, a.mi, a.mv);
  Dev<double> X((size_t)a.K * a.d + 1), ref(n), D((size_t)K1 * n), norms(K1);
  const int nblk = std::min(148, (n + 255) / 256);
  Dev<double> part((size_t)K1 * nblk);
  if (a.K)
    PE_CUDA_CHECK(cudaMemcpyAsync(X.p, a.X, sizeof(double) * a.K * a.d, cudaMemcpyHostToDevice, a.st));
  PE_CUDA_CHECK(cudaMemcpyAsync(ref.p, a.ref, sizeof(double) * n, cudaMemcpyHostToDevice, a.st));
  k_reconstruct_diff<<<(n + 7) / 8, 256, 0, a.st>>>(n, a.d, a.K, P.ptr.p, P.idx.p, P.val.p, X.p,
                                                    ref.p, D.p);
  k_mnorm_partial<<<dim3(nblk, K1), 256, 0, a.st>>>(n, M.ptr.p, M.idx.p, M.val.p, D.p, part.p);
  k_mnorm_final<<<(K1 + 127) / 128, 128, 0, a.st>>>(nblk, K1, part.p, norms.p);
  g_launches += 3;
  PE_CUDA_CHECK(cudaGetLastError());
  PE_CUDA_CHECK(cudaMemcpyAsync(a.norms_h, norms.p, sizeof(double) * K1, cudaMemcpyDeviceToHost, a.st));
  PE_CUDA_CHECK(cudaStreamSynchronize(a.st));
}

}  // namespace pe

extern "C" int pe_fine_reference_solve(int n, const int* M_ptr, const int* M_idx,
                                       const double* M_val, const int* A_ptr, const int* A_idx,
                                       const double* A_val, const double* b, const double* u0,
                                       double t_end, int n_steps, int keep_trajectory,
                                       double* states_h, float* step_ms, void* stream) {
  if (n <= 0 || n_steps <= 0 || !(t_end > 0.0) || !M_ptr || !A_ptr || !b || !states_h) {
    pe::set_error("pe_fine_reference_solve: need n > 0, n_steps > 0, t_end > 0 and buffers");
    return PE_ERR_ARG;
  }
  pe::RefSolveArgs a{n,     M_ptr,   M_idx, A_ptr, A_idx, M_val,          A_val,
                     b,     u0,      t_end, n_steps, states_h, keep_trajectory,
                     (cudaStream_t)stream, step_ms};
  return pe::fs_guard("pe_fine_reference_solve", pe::ref_solve_impl, &a);
}

extern "C" int pe_fine_solver_kind(int n, const int* M_ptr, const int* M_idx, const int* A_ptr,
                                   const int* A_idx, int* block) {
  if (n <= 0 || !M_ptr || !A_ptr) {
    pe::set_error("pe_fine_solver_kind: need n > 0 and CSR index arrays");
    return -1;
  }
  if (block) *block = 0;
  if (pe::fine_chain_applicable(n, M_ptr, M_idx, A_ptr, A_idx, block)) return 2;
  return (n >= pe::kSymMin && !getenv("PE_FINE_NO_SYM")) ? 1 : 0;
}

extern "C" int pe_relative_error_series(int n, int d, const int* P_ptr, const int* P_idx,
                                        const double* P_val, const int* M_ptr,
                                        const int* M_idx, const double* M_val,
                                        const double* ref, int K, const double* X,
                                        double* norms_h, void* stream) {
  if (n <= 0 || d < 0 || K < 0 || !P_ptr || !M_ptr || !ref || !norms_h || (K > 0 && !X)) {
    pe::set_error("pe_relative_error_series: need n > 0, K >= 0 and buffers");
    return PE_ERR_ARG;
  }
  pe::ErrArgs a{n, d, K, P_ptr, P_idx, M_ptr, M_idx, P_val, M_val, ref, X, norms_h,
                (cudaStream_t)stream};
  return pe::fs_guard("pe_relative_error_series", pe::err_impl, &a);
}
