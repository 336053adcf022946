// Fused coarse sweep + parareal correction + convergence norms (K2).
//
// One thread-block cluster per ensemble member walks the N coarse intervals
// sequentially (parareal.py:198-215; initial sweep :150-157):
//     g        = G(x_n^{k+1}) = Phi x_n^{k+1} + gvec        (stepping.py:161-176)
//     x_{n+1}  = F_hat_n + (g - G_cache_n)                    grouping kept exactly (:209)
//     G_cache_n = g
// Each CTA of the cluster owns a contiguous row slice of Phi = K_G^{-1} R_G (kept in
// shared memory when it fits) and the cluster barrier publishes x_{n+1} between steps,
// so there is no host round trip per coarse step.  The per-interval norms
// ||x_new - x_old|| and ||x_new|| (parareal.py:140-142) are reduced in a fixed order
// (lane-strided dot, xor tree, warps in index order, CTAs in rank order), so reruns
// are bitwise reproducible.

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "pe.h"
#include "pe_internal.h"

namespace cg = cooperative_groups;

namespace pe {

constexpr int COARSE_THREADS = 256;
constexpr int COARSE_WARPS = COARSE_THREADS / 32;

__device__ __forceinline__ double warp_sum_c(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct CoarseArgs {
  int d, N, cs;
  int phi_in_smem;
  const double* Phi;   // (E, d, d) row-major
  const double* gvec;  // (E, d)
  const double* X_old; // (E, N+1, d)
  const double* F_hat; // (E, N, d) or null (initial sweep)
  double* G_cache;     // (E, N, d)
  double* X_new;       // (E, N+1, d)
  double* partial;     // (E, N, cs, 2)
  double* diff;        // (E, 2)
  const int* active;   // (E) or null
};

__device__ __forceinline__ unsigned cs_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cs_map_rank(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cs_st_async(unsigned addr, double v, unsigned bar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               ::"r"(addr), "l"(__double_as_longlong(v)), "r"(bar) : "memory");
}
__device__ __forceinline__ void cs_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cs_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

// x_{n+1} rows travel point to point: each new row is pushed (st.async, 8 bytes) into
// every peer's double-buffered x with complete_tx on the peer's mbarrier; a CTA waits
// only for the d*8 bytes of the step it consumes (same protocol as recur.cu).
__global__ void __launch_bounds__(COARSE_THREADS) coarse_kernel(const __grid_constant__ CoarseArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int e = blockIdx.x / a.cs;
  const int d = a.d, N = a.N;
  const int r0 = (int)((long long)rank * d / a.cs), r1 = (int)((long long)(rank + 1) * d / a.cs);
  const int nrows = r1 - r0;
  const double* X_old = a.X_old + (long long)e * (N + 1) * d;
  double* X_new = a.X_new + (long long)e * (N + 1) * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (a.active && a.active[e] == 0) {  // converged member: iterate frozen (whole cluster)
    for (long long t = threadIdx.x; t < (long long)(N + 1) * nrows; t += COARSE_THREADS) {
      const int n = (int)(t / nrows), r = r0 + (int)(t % nrows);
      X_new[(long long)n * d + r] = X_old[(long long)n * d + r];
    }
    return;
  }

  extern __shared__ __align__(16) double sm[];
  double* xs2 = sm;                         // 2 x d
  double* wpart = xs2 + 2 * d;              // COARSE_WARPS * 2
  double* phis = wpart + 2 * COARSE_WARPS;  // nrows * d (optional)
  __shared__ __align__(8) unsigned long long mbar[2];
  const double* Phi = a.Phi + (long long)e * d * d;
  const double* gv = a.gvec + (long long)e * d;
  const double* F = a.F_hat ? a.F_hat + (long long)e * N * d : nullptr;
  double* Gc = a.G_cache + (long long)e * N * d;

  if (a.phi_in_smem) {
    const double* src = Phi + (long long)r0 * d;
    for (long long t = threadIdx.x; t < (long long)nrows * d; t += COARSE_THREADS) phis[t] = src[t];
  }
  for (int k = threadIdx.x; k < d; k += COARSE_THREADS) xs2[k] = X_old[k];
  for (int r = r0 + threadIdx.x; r < r1; r += COARSE_THREADS) X_new[r] = X_old[r];
  const unsigned bytes = (unsigned)(d * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cs_smem_u32(&mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cs_smem_u32(&mbar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();
  if (threadIdx.x == 0) {
    cs_expect(cs_smem_u32(&mbar[1]), bytes);            // x_1 (pushed at step 0)
    if (N > 2) cs_expect(cs_smem_u32(&mbar[0]), bytes);  // x_2 (pushed at step 1)
  }
  const unsigned bar0 = cs_smem_u32(&mbar[0]);
  const unsigned xs_base = cs_smem_u32(xs2);

  // per-row operands of step n (lane i <-> i-th row of the warp), fetched one step
  // ahead so their L2 latency hides under the previous step
  double nf_f = 0.0, nf_g = 0.0, nf_b = 0.0, nf_o = 0.0;
  auto prefetch = [&](int n) {
    const int rr = warp + COARSE_WARPS * lane;
    if (n < N && rr < nrows) {
      const long long o = (long long)n * d + r0 + rr;
      nf_b = gv[r0 + rr];
      nf_o = X_old[o + d];
      if (F) {
        nf_f = F[o];
        nf_g = Gc[o];
      }
    }
  };
  prefetch(0);
  for (int n = 0; n < N; ++n) {
    const int cur = n & 1;
    if (n > 0) {
      cs_wait(bar0 + 8 * cur, ((n - 1) >> 1) & 1);
      if (threadIdx.x == 0 && n + 2 < N) cs_expect(bar0 + 8 * cur, bytes);
    }
    const double* xs = xs2 + (size_t)cur * d;
    double sd = 0.0, sn = 0.0;  // this warp's partial ||x_new - x_old||^2, ||x_new||^2
    const double pf_f = nf_f, pf_g = nf_g, pf_b = nf_b, pf_o = nf_o;
    const bool push = (n + 1 < N);
    const unsigned nbar = bar0 + 8 * ((n + 1) & 1);
    const unsigned nbuf = xs_base + (unsigned)(((n + 1) & 1) * d * 8);
    int i = 0;
    for (int rr = warp; rr < nrows; rr += COARSE_WARPS, ++i) {
      const int r = r0 + rr;
      const double* row = a.phi_in_smem ? phis + (long long)rr * d : Phi + (long long)r * d;
      double acc = 0.0;
      for (int k = lane; k < d; k += 32) acc = fma(row[k], xs[k], acc);
      acc = warp_sum_c(acc);
      const long long o = (long long)n * d + r;
      double fb = __shfl_sync(0xffffffffu, pf_b, i & 31);
      double ff = __shfl_sync(0xffffffffu, pf_f, i & 31);
      double fg = __shfl_sync(0xffffffffu, pf_g, i & 31);
      double xo = __shfl_sync(0xffffffffu, pf_o, i & 31);
      if (i >= 32) {  // more rows per warp than lanes: plain loads
        fb = gv[r];
        xo = X_old[o + d];
        if (F) {
          ff = F[o];
          fg = Gc[o];
        }
      }
      // every lane holds the warp sum: compute the row's value redundantly
      const double g = acc + fb;
      const double x = F ? ff + (g - fg) : g;
      if (lane == 0) {
        Gc[o] = g;
        X_new[o + d] = x;
        const double df = x - xo;
        sd += df * df;
        sn += x * x;
      }
      if (push)  // lane q pushes row r of x_{n+1} into CTA q
        for (int q = lane; q < a.cs; q += 32)
          cs_st_async(cs_map_rank(nbuf + (unsigned)(r * 8), q), x, cs_map_rank(nbar, q));
    }
    prefetch(n + 1);
    if (lane == 0) {
      wpart[2 * warp] = sd;
      wpart[2 * warp + 1] = sn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double td = 0.0, tn = 0.0;
      for (int w = 0; w < COARSE_WARPS; ++w) {
        td += wpart[2 * w];
        tn += wpart[2 * w + 1];
      }
      double* p = a.partial + (((long long)e * N + n) * a.cs + rank) * 2;
      p[0] = td;
      p[1] = tn;
    }
    __syncthreads();  // wpart reused next step
  }
  cluster.sync();  // partials published; no CTA exits with pushes in flight

  if (rank == 0 && threadIdx.x == 0 && a.diff) {
    double md = 0.0, mn = 0.0;
    for (int n = 0; n < N; ++n) {
      const double* p = a.partial + ((long long)e * N + n) * a.cs * 2;
      double td = 0.0, tn = 0.0;
      for (int c = 0; c < a.cs; ++c) {
        td += p[2 * c];
        tn += p[2 * c + 1];
      }
      const double nd = sqrt(td), nn = sqrt(tn);
      md = (nd > md || nd != nd) ? nd : md;
      mn = (nn > mn || nn != nn) ? nn : mn;
    }
    a.diff[2 * e] = md;
    a.diff[2 * e + 1] = mn;
  }
}

// ---------------------------------------------------------------------------------------
// Large-d path (Phi slice does not fit in a cluster's shared memory, e.g. config 3 with
// d = 8192 and a 537 MB Phi): one launch per coarse step across all SMs so that the
// step streams Phi at HBM bandwidth (HBM-bound at cfg3), warp per row, four
// independent lane-strided accumulators (fixed combination order), per-block norm
// partials reduced in block order by a final kernel.
constexpr int CS_THREADS = 256;
constexpr int CS_WARPS = CS_THREADS / 32;

__global__ void __launch_bounds__(CS_THREADS)
    coarse_step_stream_kernel(int d, int n, int N, const double* __restrict__ Phi,
                              const double* __restrict__ gvec, const double* X_old,
                              const double* F_hat, double* G_cache, double* X_new,
                              double* partial, const int* active) {
  const int e = blockIdx.y;
  if (active && active[e] == 0) {
    if (n == 0) {  // frozen member: copy the whole iterate once
      const double* xo = X_old + (long long)e * (N + 1) * d;
      double* xn = X_new + (long long)e * (N + 1) * d;
      for (long long t = blockIdx.x * (long long)CS_THREADS + threadIdx.x; t < (long long)(N + 1) * d;
           t += (long long)gridDim.x * CS_THREADS)
        xn[t] = xo[t];
    }
    return;
  }
  extern __shared__ double xs[];
  const double* Xo = X_old + (long long)e * (N + 1) * d;
  double* Xn = X_new + (long long)e * (N + 1) * d;
  const double* xcur = (n == 0) ? Xo : Xn + (long long)n * d;  // x_n^{k+1} (row 0 = x_0)
  for (int k = threadIdx.x; k < d; k += CS_THREADS) xs[k] = __ldcg(xcur + k);
  if (n == 0)
    for (int r = blockIdx.x * CS_THREADS + threadIdx.x; r < d; r += gridDim.x * CS_THREADS)
      Xn[r] = Xo[r];
  __syncthreads();
  const double* Pm = Phi + (long long)e * d * d;
  const double* gv = gvec + (long long)e * d;
  const double* F = F_hat ? F_hat + (long long)e * N * d : nullptr;
  double* Gc = G_cache + (long long)e * N * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sd = 0.0, sn = 0.0;
  for (int r = blockIdx.x * CS_WARPS + warp; r < d; r += gridDim.x * CS_WARPS) {
    const double* row = Pm + (long long)r * d;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int k = lane;
    // 8 independent loads in flight per lane (HBM-bound stream of Phi)
    for (; k + 224 < d; k += 256) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(row + k + 32 * u);
      a0 = fma(v[0], xs[k], a0);
      a1 = fma(v[1], xs[k + 32], a1);
      a2 = fma(v[2], xs[k + 64], a2);
      a3 = fma(v[3], xs[k + 96], a3);
      a0 = fma(v[4], xs[k + 128], a0);
      a1 = fma(v[5], xs[k + 160], a1);
      a2 = fma(v[6], xs[k + 192], a2);
      a3 = fma(v[7], xs[k + 224], a3);
    }
    for (; k + 96 < d; k += 128) {
      a0 = fma(__ldcs(row + k), xs[k], a0);
      a1 = fma(__ldcs(row + k + 32), xs[k + 32], a1);
      a2 = fma(__ldcs(row + k + 64), xs[k + 64], a2);
      a3 = fma(__ldcs(row + k + 96), xs[k + 96], a3);
    }
    for (; k < d; k += 32) a0 = fma(__ldcs(row + k), xs[k], a0);
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const long long o = (long long)n * d + r;
      const double g = acc + gv[r];
      const double x = F ? F[o] + (g - Gc[o]) : g;
      Gc[o] = g;
      Xn[o + d] = x;
      const double df = x - Xo[o + d];
      sd += df * df;
      sn += x * x;
    }
  }
  __shared__ double wp[2 * CS_WARPS];
  if (lane == 0) {
    wp[2 * warp] = sd;
    wp[2 * warp + 1] = sn;
  }
  __syncthreads();
  if (threadIdx.x == 0 && partial) {
    double td = 0.0, tn = 0.0;
    for (int w = 0; w < CS_WARPS; ++w) {
      td += wp[2 * w];
      tn += wp[2 * w + 1];
    }
    double* p = partial + (((long long)e * N + n) * gridDim.x + blockIdx.x) * 2;
    p[0] = td;
    p[1] = tn;
  }
}

// One block per member; thread n sums interval n's block partials in block order (fixed),
// then the max over intervals is taken in a fixed smem tree (NaN propagates).
__global__ void coarse_norm_reduce_kernel(int N, int nblocks, const double* partial,
                                          double* diff, const int* active) {
  const int e = blockIdx.x;
  if (active && active[e] == 0) return;
  __shared__ double md[256], mn[256];
  double bd = 0.0, bn = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    const double* p = partial + ((long long)e * N + n) * nblocks * 2;
    double td = 0.0, tn = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      td += p[2 * b];
      tn += p[2 * b + 1];
    }
    const double nd = sqrt(td), nn = sqrt(tn);
    bd = (nd > bd || nd != nd) ? nd : bd;
    bn = (nn > bn || nn != nn) ? nn : bn;
  }
  md[threadIdx.x] = bd;
  mn[threadIdx.x] = bn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double a = md[threadIdx.x + o], b = mn[threadIdx.x + o];
      if (a > md[threadIdx.x] || a != a) md[threadIdx.x] = a;
      if (b > mn[threadIdx.x] || b != b) mn[threadIdx.x] = b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    diff[2 * e] = md[0];
    diff[2 * e + 1] = mn[0];
  }
}

int coarse_stream_blocks(int d) { return std::min(296, (d + CS_WARPS - 1) / CS_WARPS); }

static void coarse_correct_stream(int E, int d, int N, const double* Phi, const double* gvec,
                                  const double* X_old, const double* F_hat, double* G_cache,
                                  double* X_new, double* partial, double* diff,
                                  const int* active, cudaStream_t st) {
  const int nb = coarse_stream_blocks(d);
  const size_t smem = sizeof(double) * d;
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(coarse_step_stream_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (smem > 200 * 1024) throw Error{PE_ERR_ARG, "coarse state too large for one SM"};
  for (int n = 0; n < N; ++n) {
    coarse_step_stream_kernel<<<dim3(nb, E), CS_THREADS, smem, st>>>(
        d, n, N, Phi, gvec, X_old, F_hat, G_cache, X_new, partial, active);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
  }
  if (diff) {
    coarse_norm_reduce_kernel<<<E, 256, 0, st>>>(N, nb, partial, diff, active);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
  }
}

int coarse_cluster_size(int d) {
  if (d >= 256) return 16;
  if (d >= 64) return 8;
  if (d >= 16) return 4;
  return 1;
}

void coarse_correct(int E, int d, int N, const double* Phi, const double* gvec,
                    const double* X_old, const double* F_hat, double* G_cache, double* X_new,
                    double* partial, double* diff, const int* active, cudaStream_t st) {
  if (N <= 0 || d <= 0) return;
  CoarseArgs a;
  a.d = d;
  a.N = N;
  a.cs = coarse_cluster_size(d);
  const int rows_max = (d + a.cs - 1) / a.cs;
  size_t base = sizeof(double) * (2 * d + 2 * COARSE_WARPS);
  size_t with_phi = base + sizeof(double) * (size_t)rows_max * d;
  a.phi_in_smem = with_phi <= 200 * 1024;
  // Large d (Phi not smem-resident) or many members (more member clusters than fit at
  // once, ~9 clusters of 16): stream Phi from HBM, all SMs per step.
  if (!a.phi_in_smem || (long long)E * a.cs > 148) {
    coarse_correct_stream(E, d, N, Phi, gvec, X_old, F_hat, G_cache, X_new, partial, diff,
                          active, st);
    return;
  }
  size_t smem = a.phi_in_smem ? with_phi : base;
  a.Phi = Phi;
  a.gvec = gvec;
  a.X_old = X_old;
  a.F_hat = F_hat;
  a.G_cache = G_cache;
  a.X_new = X_new;
  a.partial = partial;
  a.diff = diff;
  a.active = active;
  static bool attr_done = false;
  if (!attr_done) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(coarse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       210 * 1024));
    PE_CUDA_CHECK(
        cudaFuncSetAttribute(coarse_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(E * a.cs);
  cfg.blockDim = dim3(COARSE_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, coarse_kernel, a));
  ++g_launches;
}

}  // namespace pe
