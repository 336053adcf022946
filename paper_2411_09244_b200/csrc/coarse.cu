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
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
  int phi_in_reg;      // rows per warp <= 5 and d <= 640: Phi rows in registers (no smem slice)
  const double* Phi;   // (E, d, d) row-major
  const double* gvec;  // (E, d); with a load series (E, N, d): member stride ge, step stride gn
  long long ge, gn;
  const double* X_old; // (E, N+1, d)
  const double* F_hat; // (E, N, d) or null (initial sweep)
  double* G_cache;     // (E, N, d)
  double* X_new;       // (E, N+1, d)
  double* partial;     // (E, N, cs, 2)
  double* diff;        // (E, 2)
  const int* active;   // (E) or null
  unsigned long long* trace;  // optional per-step timestamps (CTA 0, thread 0), debug only
};

__device__ __forceinline__ unsigned long long cs_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CS_TRACE(slot) \
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[slot] = cs_timer();

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

// x_{n+1} rows travel by st.async: the lane that finished a row stores it into every peer's
// next x buffer, completing on the peer's mbarrier; a CTA waits only on its own mbarrier
// and a step has no CTA barrier (round 2; round 1 staged the rows and issued one bulk
// DSMEM copy per peer behind a CTA barrier: 3.2 us per step at d = 600).  Each warp
// computes all of its rows together (independent accumulators sharing the x loads), and
// the per-warp norm partials go straight to global memory.
__device__ __forceinline__ void cs_fence_proxy() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// NK > 0: the warp's Phi rows live in REGISTERS for the whole sweep (lane l holds columns
// l, l + 32, ..., NK per row): the per-step pass over the 180 KB slice in shared memory
// (1.1 us of a 2.5 us step at d = 600) becomes RPW x NK register FMAs.  Same lane-strided k
// order and xor tree, so the sums are bitwise those of the shared-memory pass.
template <int RPW, bool PHIS, int NK = 0>  // rows per warp (max); Phi slice in shared memory
__device__ __forceinline__ void coarse_steps(const CoarseArgs& a, int rank, int e, int r0, int nrows,
                                             int ncopy, double* xs2, double* ybuf2,
                                             const double* phis, unsigned bar0, unsigned xs_base,
                                             unsigned yb_base, unsigned bytes) {
  const int d = a.d, N = a.N;
  const int xsd = 2 * ((d + 1) / 2) + 2;  // x buffer stride: even, so copies stay 16-byte aligned
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* X_old = a.X_old + (long long)e * (N + 1) * d;
  double* X_new = a.X_new + (long long)e * (N + 1) * d;
  const double* Phi = a.Phi + (long long)e * d * d;
  const double* gv = a.gvec + (long long)e * a.ge;
  const double* F = a.F_hat ? a.F_hat + (long long)e * N * d : nullptr;
  double* Gc = a.G_cache + (long long)e * N * d;
  const double* rowp[RPW];
  bool rv[RPW];
  const int wrows = nrows > warp ? (nrows - warp + COARSE_WARPS - 1) / COARSE_WARPS : 0;
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int rr = warp + COARSE_WARPS * j;
    rv[j] = rr < nrows;
    rowp[j] = PHIS ? phis + (long long)(rv[j] ? rr : 0) * d
                   : Phi + (long long)(r0 + (rv[j] ? rr : 0)) * d;
  }
  double pr[NK > 0 ? RPW : 1][NK > 0 ? NK : 1];
  if constexpr (NK > 0) {
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
      for (int i = 0; i < NK; ++i) {
        const int k = lane + 32 * i;
        pr[j][i] = (rv[j] && k < d) ? __ldg(Phi + (long long)(r0 + warp + COARSE_WARPS * j) * d + k) : 0.0;
      }
  }
  // Warps without rows neither read x nor send: they leave (with no CTA barrier in the
  // step loop a lagging idle warp could miss a whole phase of the receive barrier).  Warp 0
  // stays: its thread 0 arms the barrier and its own wait keeps it in step.
  if (wrows == 0 && warp != 0) {
    if (lane == 0)  // its norm partials are zeros
      for (int n = 0; n < N; ++n) {
        double* p = a.partial + ((((long long)e * N + n) * a.cs + rank) * COARSE_WARPS + warp) * 2;
        p[0] = 0.0;
        p[1] = 0.0;
      }
    return;
  }
  // lane j < RPW owns row warp + 8 j: its operands for step n are fetched one step ahead
  const int myrr = warp + COARSE_WARPS * lane;
  const bool mine = lane < RPW && myrr < nrows;
  double nf_f = 0.0, nf_g = 0.0, nf_b = 0.0, nf_o = 0.0;
  auto prefetch = [&](int n) {
    if (n < N && mine) {
      const long long o = (long long)n * d + r0 + myrr;
      nf_b = gv[(long long)n * a.gn + r0 + myrr];
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
    CS_TRACE(1 + 3 * n)
    if (n > 0) {
      cs_wait(bar0 + 8 * cur, ((n - 1) >> 1) & 1);
      if (threadIdx.x == 0 && n + 2 < N) cs_expect(bar0 + 8 * cur, bytes);
    }
    CS_TRACE(2 + 3 * n)
    const double* xs = xs2 + (size_t)cur * xsd;
    double acc[RPW];
#pragma unroll
    for (int j = 0; j < RPW; ++j) acc[j] = 0.0;
    // lane-strided k (lane, lane+32, ...) in order, four k per pass with all loads issued
    // before the FMAs; specialised on this warp's exact row count (warp-uniform) so that no
    // load is issued for an absent row (the pass is shared-memory-bandwidth bound)
    auto dot = [&](auto WR) {
      constexpr int W = decltype(WR)::value;
      for (int k0 = 0; k0 < d; k0 += 128) {
        double xk[4], rk[W][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + 32 * u + lane;
          xk[u] = (k < d) ? xs[k] : 0.0;
#pragma unroll
          for (int j = 0; j < W; ++j) rk[j][u] = (k < d) ? rowp[j][k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + 32 * u + lane < d)
#pragma unroll
            for (int j = 0; j < W; ++j) acc[j] = fma(rk[j][u], xk[u], acc[j]);
      }
    };
    if constexpr (NK > 0) {
#pragma unroll
      for (int i = 0; i < NK; ++i) {
        const int k = lane + 32 * i;
        if (k < d) {
          const double xk = xs[k];
#pragma unroll
          for (int j = 0; j < RPW; ++j) acc[j] = fma(pr[j][i], xk, acc[j]);
        }
      }
    } else
    switch (wrows) {
      case 0: break;
      case 1: dot(std::integral_constant<int, 1>{}); break;
      case 2: if constexpr (RPW >= 2) dot(std::integral_constant<int, 2>{}); break;
      case 3: if constexpr (RPW >= 3) dot(std::integral_constant<int, 3>{}); break;
      case 4: if constexpr (RPW >= 4) dot(std::integral_constant<int, 4>{}); break;
      case 5: if constexpr (RPW >= 5) dot(std::integral_constant<int, 5>{}); break;
      case 6: if constexpr (RPW >= 6) dot(std::integral_constant<int, 6>{}); break;
      case 7: if constexpr (RPW >= 7) dot(std::integral_constant<int, 7>{}); break;
      default: if constexpr (RPW >= 8) dot(std::integral_constant<int, 8>{}); break;
    }
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[3 * N + 4 + 2 * n] = cs_timer();
    double mya = 0.0;  // lane j keeps row j's sum
    if constexpr (RPW > 2) {
      // Folded xor tree: at levels 16 / 8 / 4 a lane keeps one row of a pair and hands the
      // other to its partner, so the RPW (<= 8) trees cost 4 + 2 + 1 + 1 + 1 shuffle-adds
      // instead of 5 RPW.  Every row is still summed over the pairs (l, l ^ 16), then
      // (l, l ^ 8), ...: the totals are bitwise those of the plain trees.
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = j < RPW ? acc[j] : 0.0;
      const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
      double w4[4], w2[2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double keep = b16 ? v[2 * q + 1] : v[2 * q], send = b16 ? v[2 * q] : v[2 * q + 1];
        w4[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double keep = b8 ? w4[2 * q + 1] : w4[2 * q], send = b8 ? w4[2 * q] : w4[2 * q + 1];
        w2[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
      double t = (b4 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? w2[0] : w2[1], 4);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      // row j's total sits in the lanes with (bit 4, bit 3, bit 2) = (j & 1, j & 2, j & 4)
      const int src = ((lane & 1) << 4) | ((lane & 2) << 2) | (lane & 4);
      mya = __shfl_sync(0xffffffffu, t, src);
      if (lane >= RPW) mya = 0.0;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < RPW; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
#pragma unroll
      for (int j = 0; j < RPW; ++j)
        if (lane == j) mya = acc[j];
    }
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[3 * N + 5 + 2 * n] = cs_timer();
    const double pf_f = nf_f, pf_g = nf_g, pf_b = nf_b, pf_o = nf_o;
    prefetch(n + 1);
    double sd = 0.0, sn = 0.0;
    double x = 0.0;
    if (mine) {
      const long long o = (long long)n * d + r0 + myrr;
      const double g = mya + pf_b;
      x = F ? pf_f + (g - pf_g) : g;  // grouping kept exactly (parareal.py:209)
      Gc[o] = g;
      X_new[o + d] = x;
      const double df = x - pf_o;
      sd = df * df;
      sn = x * x;
    }
    // x_{n+1}: row (warp + 8 j) goes from lane j to every CTA's next x buffer, lane q
    // storing to peer q (st.async completing on the peer's mbarrier).  No staging, no CTA
    // barrier: a peer's step n+2 stores into the buffer read here in step n+1 only after it
    // has received this warp's step n+1 rows, i.e. after this warp's dot products.
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[5 * N + 6 + 2 * n] = cs_timer();
    if (n + 1 < N) {
      const unsigned nbar = cs_map_rank(bar0 + 8 * ((n + 1) & 1), lane < a.cs ? lane : 0);
      const unsigned dstb =
          cs_map_rank(xs_base + (unsigned)((((n + 1) & 1) * xsd + r0) * 8), lane < a.cs ? lane : 0);
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const double v = __shfl_sync(0xffffffffu, x, j);
        const int rr = warp + COARSE_WARPS * j;
        if (rr < nrows && lane < a.cs) cs_st_async(dstb + (unsigned)(rr * 8), v, nbar);
      }
    }
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[5 * N + 7 + 2 * n] = cs_timer();
    // per-warp norm partials, summed later in (rank, warp) order
    // only lanes < RPW (<= 8) hold non-zero squares: the levels 16 and 8 would add +0.0
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
      sn += __shfl_xor_sync(0xffffffffu, sn, o);
    }
    if (lane == 0) {
      double* p = a.partial + ((((long long)e * N + n) * a.cs + rank) * COARSE_WARPS + warp) * 2;
      p[0] = sd;
      p[1] = sn;
    }
    CS_TRACE(3 + 3 * n)
  }
}

__global__ void __launch_bounds__(COARSE_THREADS, 1) coarse_kernel(const __grid_constant__ CoarseArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int e = blockIdx.x / a.cs;
  const int d = a.d, N = a.N;
  const int half = (d + 1) / 2;  // row pairs
  const int p0 = (int)((long long)rank * half / a.cs), p1 = (int)((long long)(rank + 1) * half / a.cs);
  const int r0 = 2 * p0, r1 = min(d, 2 * p1);
  const int nrows = max(0, r1 - r0), ncopy = 2 * (p1 - p0);
  const double* X_old = a.X_old + (long long)e * (N + 1) * d;
  double* X_new = a.X_new + (long long)e * (N + 1) * d;

  if (a.active && a.active[e] == 0) {  // converged member: iterate frozen (whole cluster)
    for (long long t = threadIdx.x; t < (long long)(N + 1) * nrows; t += COARSE_THREADS) {
      const int n = (int)(t / nrows), r = r0 + (int)(t % nrows);
      X_new[(long long)n * d + r] = X_old[(long long)n * d + r];
    }
    return;
  }

  extern __shared__ __align__(16) double sm[];
  const int xsd = 2 * half + 2;                // even stride: 16-byte aligned copies
  double* xs2 = sm;                            // 2 x xsd
  double* ybuf2 = xs2 + 2 * xsd;               // 2 x ncopy_max
  const int ncmax = 2 * ((half + a.cs - 1) / a.cs);
  double* phis = ybuf2 + 2 * ncmax;            // nrows * d (optional)
  __shared__ __align__(8) unsigned long long mbar[2];
  const double* Phi = a.Phi + (long long)e * d * d;

  if (a.phi_in_smem && !a.phi_in_reg) {
    // slice -> smem by 16-byte cp.async (no register staging: the staged scalar copy is a
    // latency-bound loop that costs tens of us per cluster, once per member of an ensemble)
    const double* src = Phi + (long long)r0 * d;
    const long long tot = (long long)nrows * d;
    if (((reinterpret_cast<unsigned long long>(src) | (unsigned long long)cs_smem_u32(phis)) & 15) == 0) {
      for (long long t = 2LL * threadIdx.x; t + 1 < tot; t += 2LL * COARSE_THREADS)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(cs_smem_u32(phis + t)),
                     "l"(src + t));
      if ((tot & 1) && threadIdx.x == 0) phis[tot - 1] = src[tot - 1];
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else {
      for (long long t = threadIdx.x; t < tot; t += COARSE_THREADS) phis[t] = src[t];
    }
  }
  for (int k = threadIdx.x; k < 2 * xsd; k += COARSE_THREADS) xs2[k] = (k < d) ? X_old[k] : 0.0;
  for (int k = threadIdx.x; k < 2 * ncmax; k += COARSE_THREADS) ybuf2[k] = 0.0;  // pad rows
  for (int r = r0 + threadIdx.x; r < r1; r += COARSE_THREADS) X_new[r] = X_old[r];
  const unsigned bytes = (unsigned)(d * 8);  // every row of x_{n+1}, from all CTAs
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
  const unsigned xs_base = cs_smem_u32(xs2), yb_base = cs_smem_u32(ybuf2);
  const int rpw = (nrows + COARSE_WARPS - 1) / COARSE_WARPS;
  auto run = [&](auto R, auto S) {
    coarse_steps<decltype(R)::value, decltype(S)::value>(a, rank, e, r0, nrows, ncopy, xs2, ybuf2,
                                                          phis, bar0, xs_base, yb_base, bytes);
  };
  using T1 = std::true_type;
  using F1 = std::false_type;
  if (a.phi_in_reg)
    coarse_steps<5, false, 20>(a, rank, e, r0, nrows, ncopy, xs2, ybuf2, phis, bar0, xs_base, yb_base,
                               bytes);
  else if (rpw <= 1)
    a.phi_in_smem ? run(std::integral_constant<int, 1>{}, T1{}) : run(std::integral_constant<int, 1>{}, F1{});
  else if (rpw <= 2)
    a.phi_in_smem ? run(std::integral_constant<int, 2>{}, T1{}) : run(std::integral_constant<int, 2>{}, F1{});
  else if (rpw <= 4)
    a.phi_in_smem ? run(std::integral_constant<int, 4>{}, T1{}) : run(std::integral_constant<int, 4>{}, F1{});
  else
    a.phi_in_smem ? run(std::integral_constant<int, 8>{}, T1{}) : run(std::integral_constant<int, 8>{}, F1{});
  cluster.sync();  // partials published; no CTA exits with copies in flight

  if (rank == 0 && a.diff) {
    // thread n sums interval n's (rank, warp) partials in order; max over intervals in a
    // fixed smem tree (NaN propagates)
    __shared__ double rd[COARSE_THREADS], rn[COARSE_THREADS];
    const int nb = a.cs * COARSE_WARPS;
    double md = 0.0, mn = 0.0;
    for (int n = threadIdx.x; n < N; n += COARSE_THREADS) {
      const double* p = a.partial + ((long long)e * N + n) * nb * 2;
      double td = 0.0, tn = 0.0;
      for (int c = 0; c < nb; ++c) {
        td += p[2 * c];
        tn += p[2 * c + 1];
      }
      const double nd = sqrt(td), nn = sqrt(tn);
      md = (nd > md || nd != nd) ? nd : md;
      mn = (nn > mn || nn != nn) ? nn : mn;
    }
    rd[threadIdx.x] = md;
    rn[threadIdx.x] = mn;
    __syncthreads();
    for (int o = COARSE_THREADS / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) {
        const double x = rd[threadIdx.x + o], y = rn[threadIdx.x + o];
        if (x > rd[threadIdx.x] || x != x) rd[threadIdx.x] = x;
        if (y > rn[threadIdx.x] || y != y) rn[threadIdx.x] = y;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      a.diff[2 * e] = rd[0];
      a.diff[2 * e + 1] = rn[0];
    }
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
int coarse_stream_blocks(int d) { return std::min(296, (d + CS_WARPS - 1) / CS_WARPS); }

__global__ void __launch_bounds__(CS_THREADS)
    coarse_step_stream_kernel(int d, int n, int N, const double* __restrict__ Phi,
                              const double* __restrict__ gvec, long long ge, long long gn,
                              const double* X_old,
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
  const double* gv = gvec + (long long)e * ge + (long long)n * gn;
  const double* F = F_hat ? F_hat + (long long)e * N * d : nullptr;
  double* Gc = G_cache + (long long)e * N * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sd = 0.0, sn = 0.0;
  for (int r = blockIdx.x * CS_WARPS + warp; r < d; r += gridDim.x * CS_WARPS) {
    const double* row = Pm + (long long)r * d;
    // the epilogue's operands are loaded ahead of the row so that their latency overlaps
    // the stream (left to the compiler, they were serialised after it in some builds:
    // 45 vs 105 us per cfg4 coarse step)
    const long long o = (long long)n * d + r;
    double pg = 0.0, pf = 0.0, pc = 0.0, px = 0.0;
    if (lane == 0) {
      pg = gv[r];
      px = Xo[o + d];
      if (F) {
        pf = F[o];
        pc = Gc[o];
      }
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int k = lane;
    // 16 (then 8, 4) independent loads in flight per lane (HBM-bound stream of Phi)
#pragma unroll 1
    for (; k + 480 < d; k += 512) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcs(row + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 16; u += 4) {
        a0 = fma(v[u], xs[k + 32 * u], a0);
        a1 = fma(v[u + 1], xs[k + 32 * u + 32], a1);
        a2 = fma(v[u + 2], xs[k + 32 * u + 64], a2);
        a3 = fma(v[u + 3], xs[k + 32 * u + 96], a3);
      }
    }
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
    // tail: element k + 32 u still goes to accumulator u % 4 (the bulk kernel's order)
    if (k < d) a0 = fma(__ldcs(row + k), xs[k], a0);  // at most three strides remain
    if (k + 32 < d) a1 = fma(__ldcs(row + k + 32), xs[k + 32], a1);
    if (k + 64 < d) a2 = fma(__ldcs(row + k + 64), xs[k + 64], a2);
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double g = acc + pg;
      const double x = F ? pf + (g - pc) : g;
      Gc[o] = g;
      Xn[o + d] = x;
      const double df = x - px;
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


static void coarse_correct_stream(int E, int d, int N, const double* Phi, const double* gvec,
                                  long long ge, long long gn,
                                  const double* X_old, const double* F_hat, double* G_cache,
                                  double* X_new, double* partial, double* diff,
                                  const int* active, cudaStream_t st) {
  // Ensembles: about one resident wave of CTAs (8 per SM) over all members, several rows
  // per warp.  One row per warp in 4800 short-lived CTAs reloaded the member's state for 8
  // rows each: 43.7 us per cfg4 coarse step, 5.21 ms per iteration; measured per blocks
  // per member (tools sweep, PE_CS_BLOCKS): 38: 5.12, 25: 5.06, 19: 4.99, 15: 5.16,
  // 13: 4.94, 10: 5.13 ms
  int nb = coarse_stream_blocks(d);
  if (E > 1) nb = std::min(nb, std::max(1, (148 * 8 + E / 2) / E));  // one resident wave
  if (getenv("PE_CS_BLOCKS")) nb = std::max(1, std::min(296, atoi(getenv("PE_CS_BLOCKS"))));
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
        d, n, N, Phi, gvec, ge, gn, X_old, F_hat, G_cache, X_new, partial, active);
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
                    double* partial, double* diff, const int* active, cudaStream_t st,
                    const double* gseries) {
  // gseries (E, N, d): per-step load terms K_G^-1 f(t_n + Dt) (time-dependent loads)
  const long long ge = gseries ? (long long)N * d : d, gn = gseries ? d : 0;
  if (gseries) gvec = gseries;
  if (N <= 0 || d <= 0) return;
  CoarseArgs a;
  a.d = d;
  a.N = N;
  a.cs = coarse_cluster_size(d);
  const int half = (d + 1) / 2;
  const int rows_max = 2 * ((half + a.cs - 1) / a.cs);
  size_t base = sizeof(double) * (2 * (size_t)(2 * half + 2) + 2 * (size_t)rows_max);
  size_t with_phi = base + sizeof(double) * (size_t)rows_max * d;
  a.phi_in_smem = with_phi <= 200 * 1024;
  static const bool no_reg = getenv("PE_COARSE_NO_REG") != nullptr;
  // (3 or more rows per warp: below that the shared-memory pass is short anyway)
  a.phi_in_reg = !no_reg && a.phi_in_smem && d <= 640 && rows_max <= 5 * COARSE_WARPS &&
                 rows_max > 2 * COARSE_WARPS;
  // Large d (Phi not smem-resident): stream Phi from HBM, all SMs per step.  Ensembles with
  // more member clusters than fit at once (~7-9 clusters of 16) also run here: the hardware
  // schedules the member clusters in waves, each keeps its member's Phi in shared memory for
  // all N steps, so Phi comes from HBM once per sweep instead of once per step.  Measured at
  // cfg4 (64 members, d = 600, N = 32): 0.72 ms per sweep against 1.07 ms for the per-step
  // stream over all members (4.66 vs 5.00 ms per iteration); PE_COARSE_ENS_STREAM=1 restores
  // the stream.
  static const bool ens_stream = getenv("PE_COARSE_ENS_STREAM") != nullptr;
  if (!a.phi_in_smem || ((long long)E * a.cs > 148 && ens_stream)) {
    coarse_correct_stream(E, d, N, Phi, gvec, ge, gn, X_old, F_hat, G_cache, X_new, partial, diff,
                          active, st);
    return;
  }
  size_t smem = (a.phi_in_smem && !a.phi_in_reg) ? with_phi : base;
  a.Phi = Phi;
  a.gvec = gvec;
  a.ge = ge;
  a.gn = gn;
  a.X_old = X_old;
  a.F_hat = F_hat;
  a.G_cache = G_cache;
  a.X_new = X_new;
  a.partial = partial;
  a.diff = diff;
  a.active = active;
  static const bool trace = getenv("PE_COARSE_TRACE") != nullptr;
  a.trace = nullptr;
  if (trace) {
    PE_CUDA_CHECK(cudaMalloc(&a.trace, sizeof(unsigned long long) * (7 * N + 10)));
    PE_CUDA_CHECK(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * (7 * N + 10), st));
  }
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
  if (trace) {
    std::vector<unsigned long long> h(7 * N + 10);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    PE_CUDA_CHECK(cudaMemcpy(h.data(), a.trace, sizeof(unsigned long long) * h.size(),
                             cudaMemcpyDeviceToHost));
    double w = 0, cmp = 0, rest = 0, dot = 0, shf = 0, xc = 0, snd = 0, nrm = 0;
    for (int n = 0; n < N; ++n) {
      dot += (h[3 * N + 4 + 2 * n] - h[2 + 3 * n]) * 1e-3;
      shf += (h[3 * N + 5 + 2 * n] - h[3 * N + 4 + 2 * n]) * 1e-3;
      xc += (h[5 * N + 6 + 2 * n] - h[3 * N + 5 + 2 * n]) * 1e-3;
      snd += (h[5 * N + 7 + 2 * n] - h[5 * N + 6 + 2 * n]) * 1e-3;
      nrm += (h[3 + 3 * n] - h[5 * N + 7 + 2 * n]) * 1e-3;
      w += (h[2 + 3 * n] - h[1 + 3 * n]) * 1e-3;
      cmp += (h[3 + 3 * n] - h[2 + 3 * n]) * 1e-3;
      if (n + 1 < N) rest += (h[1 + 3 * (n + 1)] - h[3 + 3 * n]) * 1e-3;
    }
    fprintf(stderr, "coarse trace (d=%d cs=%d): per step wait %.3f compute %.3f (dot %.3f shfl %.3f"
            " x %.3f send %.3f norms %.3f) copy %.3f us\n", d, a.cs, w / N, cmp / N, dot / N, shf / N,
            xc / N, snd / N, nrm / N, rest / N);
    cudaFree(a.trace);
  }
}

}  // namespace pe
