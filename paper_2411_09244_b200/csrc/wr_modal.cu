// Modal waveform relaxation: the all-at-once WR sweep (allatonce.py:220-298) carried out in
// the generalized eigenbases of the pencils (A11, M11) and (A22, M22).
//
// With A11 V1 = M11 V1 diag(mu1), V1^T M11 V1 = I (likewise V2 for the w block), y = V1^-1 u
// and z = V2^-1 w, one sweep of the reference becomes
//   rhs   r~_s = [-V1^T A12 V2 | -V1^T M12 V2 / dt] [z_s ; z_s - z_{s-1}] + V1^T f1
//               + [s = 0] (y0 - alpha y_J^prev) / dt                         (build_rhs)
//   u     (B + mu1_i) y_i = r~_i for every mode i: B is the alpha-corner bidiagonal time
//         matrix of TimeMatrixB (allatonce.py:36-67), so the shifted solves that
//         ImplicitAllAtOnce performs by diagonalising B (:100-133) reduce to one scalar
//         recurrence per (mode, interval) plus its corner closure:
//           y_s = a (y_{s-1} + dt r_s),  y_0 = a (alpha y_{J-1} + dt r_0),  a = 1/(1 + mu dt)
//           => y_0 = a (alpha c + dt r_0) / (1 - alpha a^J),  c = sum_{s>=1} a^{J-s} dt r_s
//   w     h_s = dt V2^T (f2 - M12^T du_s - A12^T u_s),  z_{s+1} = lam z_s + h_s,
//         lam = 1 - dt mu2                                                      (_w_sweep)
//   norms ||U_new,s - U_s|| = ||V1 (Y_new,s - Y_s)||, likewise W             (:250-254)
// The two contractions (rhs, h) and the norm products are DMMA GEMMs (gemm_f64.cu); the
// time recurrences are the elementwise scans below.  libpe runs the scans in place (Yc == Yn,
// Zc == Zn: every thread reads an element before it overwrites it) and they skip stopped
// intervals, so a stopped interval keeps the waveforms of its last sweep with no commit copy.
//
// Layout per member: Y = [y0, y0, Y_0 .. Y_{J-1}] as J+2 blocks of a (d1 x nc)
// column-major matrix (L1 = d1 nc); Z likewise with d2.  DY, DZ, EY, EZ, R, H: J blocks.

#include <cmath>

#include "pe.h"
#include "pe_internal.h"
#include "wr_stop.cuh"

namespace pe {

static int grid_1d(long long n, int threads) {
  return (int)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 148 * 16));
}

// Seeds (allatonce.py:239-241): U = u0, W = w0 on every row, u_J^prev = u0; DZ = 0.
// Y0 / Z0 hold V^-1 u0 / V^-1 w0 per (member, interval).  Buffer 0 is the first sweep's
// "current" buffer: all of its blocks are seeded; buffer 1 gets the two seed blocks.
__global__ void modal_seed_kernel(int E, int nc, int d1, int d2, int J,
                                  const double* __restrict__ Y0, const double* __restrict__ Z0,
                                  double* Yb0, double* Yb1, double* Zb0, double* Zb1, double* DZ) {
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const long long tu = (long long)E * L1, total = tu + (long long)E * L2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < tu) {
      const int e = (int)(t / L1);
      const long long r = t - e * L1;
      const double y = Y0[t];
      double* a = Yb0 + (long long)e * (J + 2) * L1 + r;
      double* b = Yb1 + (long long)e * (J + 2) * L1 + r;
      for (int k = 0; k < J + 2; ++k) a[k * L1] = y;
      if (Yb1) {
        b[0] = y;
        b[L1] = y;
      }
    } else {
      const long long q = t - tu;
      const int e = (int)(q / L2);
      const long long r = q - e * L2;
      const double z = Z0[q];
      double* a = Zb0 + (long long)e * (J + 2) * L2 + r;
      double* b = Zb1 + (long long)e * (J + 2) * L2 + r;
      for (int k = 0; k < J + 2; ++k) a[k * L2] = z;
      if (Zb1) {
        b[0] = z;
        b[L2] = z;
      }
      double* dz = DZ + (long long)e * J * L2 + r;
      for (int k = 0; k < J; ++k) dz[k * L2] = 0.0;
    }
  }
}

void modal_seed(int E, int nc, int d1, int d2, int J, const double* Y0, const double* Z0,
                double* Yb0, double* Yb1, double* Zb0, double* Zb1, double* DZ, cudaStream_t st) {
  const long long total = (long long)E * nc * (d1 + d2);
  if (total == 0) return;
  modal_seed_kernel<<<grid_1d(total, 256), 256, 0, st>>>(E, nc, d1, d2, J, Y0, Z0, Yb0, Yb1, Zb0,
                                                         Zb1, DZ);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// Software-pipelined time walk for the scans: the loads of chunk c+1 (MSCAN_DEPTH steps of
// one or two J-block arrays) are in flight while chunk c is consumed, so a thread keeps
// ~2 x MSCAN_DEPTH loads outstanding for the whole walk (one chain per thread is all the
// parallelism there is: E x d x nc chains).
constexpr int MSCAN_DEPTH = 8;
template <bool TWO, class Step>
__device__ __forceinline__ void scan_walk(int s_begin, int J, long long stride,
                                          const double* __restrict__ a, long long a_off,
                                          const double* __restrict__ b, long long b_off, Step&& step) {
  double va[MSCAN_DEPTH], wa[MSCAN_DEPTH], vb[MSCAN_DEPTH], wb[MSCAN_DEPTH];
  auto load = [&](double (&v)[MSCAN_DEPTH], double (&w)[MSCAN_DEPTH], int s0) {
#pragma unroll
    for (int q = 0; q < MSCAN_DEPTH; ++q)
      if (s0 + q < J) {
        v[q] = a[(long long)(s0 + q + a_off) * stride];
        if (TWO) w[q] = b[(long long)(s0 + q + b_off) * stride];
      }
  };
  auto run = [&](const double (&v)[MSCAN_DEPTH], const double (&w)[MSCAN_DEPTH], int s0) {
#pragma unroll
    for (int q = 0; q < MSCAN_DEPTH; ++q)
      if (s0 + q < J) step(s0 + q, v[q], TWO ? w[q] : 0.0);
  };
  load(va, wa, s_begin);
  for (int s0 = s_begin; s0 < J; s0 += 2 * MSCAN_DEPTH) {
    load(vb, wb, s0 + MSCAN_DEPTH);
    run(va, wa, s0);
    load(va, wa, s0 + 2 * MSCAN_DEPTH);
    run(vb, wb, s0 + MSCAN_DEPTH);
  }
}

// u solve in modal coordinates: one thread per (member, mode i, interval n).
// In:  R (J blocks, r~ without the row-0 term), Yc (current buffer).
// Out: Yn blocks 2..J+1, DY (lagged du of _w_sweep: DY_s = Ux[s+1] - Ux[s] with
//      Ux = [y0, y0, Y_0, ..]), EY = Y_new - Y_cur (the update whose norm is the residual).
__global__ void modal_uscan_kernel(int nc, int d1, int J, int E, double dt, double alpha,
                                   const double* __restrict__ acoef,
                                   const double* __restrict__ cden, const double* __restrict__ R,
                                   const double* Yc, double* Yn,  // may alias (in place)
                                   double* __restrict__ DY, double* __restrict__ EY,
                                   const WrColumnState* __restrict__ cs) {
  pdl_enter();
  const long long L1 = (long long)d1 * nc;
  const long long total = (long long)E * L1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / L1);
    const long long r = t - e * L1;
    const int n = (int)(r / d1), i = (int)(r - (long long)n * d1);
    if (!cs[(long long)e * nc + n].active) continue;
    const double a = acoef[(long long)e * d1 + i], cd = cden[(long long)e * d1 + i];
    const double* rp = R + (long long)e * J * L1 + r;
    const double* yc = Yc + (long long)e * (J + 2) * L1 + r;
    double* yn = Yn + (long long)e * (J + 2) * L1 + r;
    double* dy = DY + (long long)e * J * L1 + r;
    double* ey = EY + (long long)e * J * L1 + r;
    const double y0 = yc[0], yJ = yc[(long long)(J + 1) * L1];
    // pass 1: c = sum_{s=1}^{J-1} a^{J-s} dt r_s
    double c = 0.0;
    scan_walk<false>(1, J, L1, rp, 0, rp, 0, [&](int, double v, double) { c = a * fma(dt, v, c); });
    const double r0 = rp[0] + (y0 - alpha * yJ) / dt;
    double y = a * fma(alpha, c, dt * r0) * cd;
    // pass 2: y_s = a (y_{s-1} + dt r_s)
    double p1 = y0, p2 = y0;  // Y_{s-1}, Y_{s-2}
    scan_walk<true>(0, J, L1, rp, 0, yc, 2, [&](int s, double v, double w) {
      if (s > 0) y = a * fma(dt, v, y);
      yn[(long long)(s + 2) * L1] = y;
      ey[(long long)s * L1] = y - w;
      dy[(long long)s * L1] = p1 - p2;
      p2 = p1;
      p1 = y;
    });
  }
}

void modal_uscan(int E, int nc, int d1, int J, double dt, double alpha, const double* acoef,
                 const double* cden, const double* R, const double* Yc, double* Yn, double* DY,
                 double* EY, const WrColumnState* cs, cudaStream_t st) {
  const long long total = (long long)E * d1 * nc;
  if (total == 0 || J == 0) return;
  launch_k(modal_uscan_kernel, dim3(grid_1d(total, 64)), dim3(64), 0, st, nc, d1, J, E, dt, alpha,
           acoef, cden, R, Yc, Yn, DY, EY, cs);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// w recursion in modal coordinates: z_{s+1} = lam z_s + h_s from z_{-1} = z0 (block 1).
// Out: Zn blocks 2..J+1, DZ (the next sweep's build_rhs difference: DZ_s = Z_{s-1} - Z_{s-2},
//      Z_{-1} = Z_{-2} = z0), EZ = Z_new - Z_cur.
__global__ void modal_wscan_kernel(int nc, int d2, int J, int E, const double* __restrict__ lam,
                                   const double* __restrict__ H, const double* Zc,
                                   double* Zn, double* __restrict__ DZ,  // Zc, Zn may alias
                                   double* __restrict__ EZ, const WrColumnState* __restrict__ cs) {
  pdl_enter();
  const long long L2 = (long long)d2 * nc;
  const long long total = (long long)E * L2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / L2);
    const long long r = t - e * L2;
    const int n = (int)(r / d2), i = (int)(r - (long long)n * d2);
    if (!cs[(long long)e * nc + n].active) continue;
    const double l = lam[(long long)e * d2 + i];
    const double* hp = H + (long long)e * J * L2 + r;
    const double* zc = Zc + (long long)e * (J + 2) * L2 + r;
    double* zn = Zn + (long long)e * (J + 2) * L2 + r;
    double* dz = DZ + (long long)e * J * L2 + r;
    double* ez = EZ + (long long)e * J * L2 + r;
    double z = zc[L2];
    double p1 = z, p2 = z;
    scan_walk<true>(0, J, L2, hp, 0, zc, 2, [&](int s, double v, double w) {
      z = fma(l, z, v);
      zn[(long long)(s + 2) * L2] = z;
      ez[(long long)s * L2] = z - w;
      dz[(long long)s * L2] = p1 - p2;
      p2 = p1;
      p1 = z;
    });
  }
}

void modal_wscan(int E, int nc, int d2, int J, const double* lam, const double* H,
                 const double* Zc, double* Zn, double* DZ, double* EZ, const WrColumnState* cs,
                 cudaStream_t st) {
  const long long total = (long long)E * d2 * nc;
  if (total == 0 || J == 0) return;
  launch_k(modal_wscan_kernel, dim3(grid_1d(total, 64)), dim3(64), 0, st, nc, d2, J, E, lam, H, Zc,
           Zn, DZ, EZ, cs);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// Stop decision.  Phase 1, one thread per (side, member, column (s, n)):
// ||dU_s|| = sqrt(sum of the norm GEMM's 8-row block partials, blocks in ascending order),
// max over s by an atomic max on the IEEE bits (exact and order-free for the non-negative
// norms; NaN / inf propagate as the largest bit patterns).  Phase 2, the last CTA (ticket):
// residual = max_s ||dU_s|| + max_s ||dW_s|| (allatonce.py:250-254) and the reference stop
// tests per interval; it also re-zeroes the maxima and the ticket for the next sweep.
constexpr int DECIDE_THREADS = 256;
__global__ void __launch_bounds__(DECIDE_THREADS)
    modal_decide_kernel(int E, int nc, int d1, int d2, int J, const double* __restrict__ nu,
                        long long nu_g, long long nu_m, const double* __restrict__ nw,
                        long long nw_g, long long nw_m, unsigned long long* colmax,
                        unsigned* ticket, WrColumnState* cs, double tol, int max_iter,
                        double* resid_hist, int* active_count, int par_new,
                        cudaGraphConditionalHandle cond, int use_cond) {
  pdl_enter();
  const long long NJ = (long long)J * nc, per = (long long)E * NJ;
  const int gu = (d1 + 7) / 8, gw = (d2 + 7) / 8;
  // four lanes per column: lane q sums the blocks g = q, q+4, ... in ascending order,
  // then ((s0 + s1) + (s2 + s3)) by shuffles (fixed order: deterministic)
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long col = t >> 2;
  const int q = (int)(t & 3);
  double acc = 0.0;
  bool live = false;
  int side = 0, e = 0, n = 0;
  if (col < 2 * per) {
    side = (int)(col / per);
    const long long rem = col - side * per;
    e = (int)(rem / NJ);
    const long long j = rem - e * NJ;
    n = (int)(j % nc);
    const int G = side ? gw : gu;
    live = G > 0 && cs[(long long)e * nc + n].active;
    if (live) {
      const double* p = side ? nw + e * nw_m + j : nu + e * nu_m + j;
      const long long gs = side ? nw_g : nu_g;
#pragma unroll 4
      for (int g = q; g < G; g += 4) acc += p[g * gs];
    }
  }
  const double a1 = __shfl_down_sync(0xffffffffu, acc, 1);
  acc += a1;  // lanes q = 0, 2 now hold s0 + s1, s2 + s3
  const double a2 = __shfl_down_sync(0xffffffffu, acc, 2);
  if (live && q == 0)
    atomicMax(colmax + (long long)side * E * nc + (long long)e * nc + n,
              (unsigned long long)__double_as_longlong(sqrt(acc + a2)));
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;
  const long long ncs = (long long)E * nc;
  int still = 0;  // intervals that keep iterating (written, not accumulated: no memset)
  for (long long base = 0; base < ncs; base += blockDim.x) {
    const long long en = base + threadIdx.x;
    bool go = false;
    if (en < ncs && cs[en].active) {
    WrColumnState c = cs[en];
    const double mu = __longlong_as_double((long long)__ldcg(colmax + en));
    const double mw = __longlong_as_double((long long)__ldcg(colmax + ncs + en));
    colmax[en] = 0ull;
    colmax[ncs + en] = 0ull;
    double resid = 0.0;
    if (d1 > 0) resid += mu;
    if (d2 > 0) resid += mw;
    c.fpar = par_new;  // this sweep wrote the interval's latest waveforms
    go = wr_stop_update(c, resid, tol, max_iter, resid_hist ? resid_hist + en * max_iter : nullptr);
    cs[en] = c;
    }
    still += __syncthreads_count(go);
  }
  if (threadIdx.x == 0) {
    *active_count = still;
    // device-side sweep loop (pe_api.cu run_sweeps): the enclosing while-node of the
    // captured graph runs another sweep only while some interval is still iterating
    if (use_cond) {
      active_count[2] += 1;  // counter slot 2 (loop mode runs buffer parity 0): sweeps run
      cudaGraphSetConditional(cond, still > 0 ? 1u : 0u);
    }
  }
}

void modal_decide(int E, int nc, int d1, int d2, int J, const double* nu, long long nu_g,
                  long long nu_m, const double* nw, long long nw_g, long long nw_m,
                  unsigned long long* colmax, unsigned* ticket, WrColumnState* cs, double tol,
                  int max_iter, double* resid_hist, int* active_count, int par_new,
                  cudaStream_t st, cudaGraphConditionalHandle cond, int use_cond) {
  const long long total = 8LL * E * J * nc;  // four lanes per (side, member, column)
  const int blocks = (int)std::max<long long>(1, (total + DECIDE_THREADS - 1) / DECIDE_THREADS);
  launch_k(modal_decide_kernel, dim3(blocks), dim3(DECIDE_THREADS), 0, st, E, nc, d1, d2, J, nu,
           nu_g, nu_m, nw, nw_g, nw_m, colmax, ticket, cs, tol, max_iter, resid_hist, active_count,
           par_new, cond, use_cond);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe

namespace pe {

__global__ void wr_state_init_kernel(long long ncs, WrColumnState* cs, double* resid_hist,
                                     int max_iter) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncs;
       t += (long long)gridDim.x * blockDim.x) {
    WrColumnState s;
    s.active = 1;
    s.iterations = 0;
    s.stall = 0;
    s.reason = PE_STOP_MAX_ITER;
    s.prev = INFINITY;
    s.r0 = 0.0;
    s.fpar = 0;
    s.pad = 0;
    cs[t] = s;
  }
  if (resid_hist)
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncs * max_iter;
         t += (long long)gridDim.x * blockDim.x)
      resid_hist[t] = NAN;
}

void wr_state_init(long long ncs, WrColumnState* cs, double* resid_hist, int max_iter,
                   cudaStream_t st) {
  wr_state_init_kernel<<<grid_1d(ncs * std::max(1, max_iter), 256), 256, 0, st>>>(ncs, cs, resid_hist,
                                                                               max_iter);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe
