// Waveform-relaxation bookkeeping kernels (allatonce.py:232-298): per-interval seeds,
// the backward difference of the new u waveform, the masked commit with the
// reference's residual / stop logic, and the final-state gather.
//
// Waveform layout per member: Ux = [u0, u0, U_0 .. U_{J-1}] as J+2 blocks of a
// (d1 x ncols) column-major matrix (block b, column n at b*L1 + n*d1, L1 = d1*ncols);
// Wx likewise with d2.  Blocks 0,1 are the lag/start seeds (allatonce.py:154,222).

#include <cmath>

#include "pe.h"
#include "pe_internal.h"
#include "wr_stop.cuh"

namespace pe {

__global__ void wr_init_kernel(int E, int nc, int d1, int d2, int J, double alpha,
                               const double* __restrict__ X, double* Ux_cur, double* Ux_new,
                               double* Wx_cur, double* Wx_new, double* V, WrColumnState* cs,
                               double* resid_hist, int max_iter) {
  const int d = d1 + d2;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const long long total = (long long)E * nc * d;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t % d);
    const long long en = t / d;  // e*nc + n
    const int n = (int)(en % nc);
    const int e = (int)(en / nc);
    const double x = X[t];
    if (r < d1) {
      double* uc = Ux_cur + (long long)e * (J + 2) * L1 + (long long)n * d1 + r;
      double* un = Ux_new + (long long)e * (J + 2) * L1 + (long long)n * d1 + r;
      for (int b = 0; b < J + 2; ++b) uc[b * L1] = x;  // U rows seeded with u0 (:239)
      un[0] = x;
      un[L1] = x;
      // u_start - alpha * u_final_prev with u_final_prev = u0 (:157, :241)
      V[(long long)e * L1 + (long long)n * d1 + r] = x - alpha * x;
    } else {
      const int q = r - d1;
      double* wc = Wx_cur + (long long)e * (J + 2) * L2 + (long long)n * d2 + q;
      double* wn = Wx_new + (long long)e * (J + 2) * L2 + (long long)n * d2 + q;
      for (int b = 0; b < J + 2; ++b) wc[b * L2] = x;  // W rows seeded with w0 (:240)
      wn[0] = x;
      wn[L2] = x;
    }
  }
  const long long ncs = (long long)E * nc;
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
  if (resid_hist) {
    const long long nh = ncs * max_iter;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nh;
         t += (long long)gridDim.x * blockDim.x)
      resid_hist[t] = NAN;
  }
}

void wr_init(int E, int nc, int d1, int d2, int J, double alpha, const double* X_in,
             double* Ux_cur, double* Ux_new, double* Wx_cur, double* Wx_new, double* V,
             WrColumnState* cs, double* resid_hist, int max_iter, cudaStream_t st) {
  long long total = (long long)E * nc * (d1 + d2);
  int blocks = (int)std::min<long long>((total + 255) / 256 + 1, 148 * 8);
  wr_init_kernel<<<blocks, 256, 0, st>>>(E, nc, d1, d2, J, alpha, X_in, Ux_cur, Ux_new, Wx_cur,
                                         Wx_new, V, cs, resid_hist, max_iter);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// DU_s = Ux[s+1] - Ux[s], s = 0..J-1: the (u_hist[1:] - u_hist[:-1]) of _w_sweep
// (allatonce.py:222-223) without the 1/dt, which is folded into the operator.
__global__ void wr_diff_u_kernel(long long L1, int J, int E, const double* __restrict__ Ux,
                                 double* __restrict__ DU) {
  const long long per = (long long)J * L1;
  const long long total = per * E;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / per);
    const long long r = t - e * per;  // s*L1 + l
    const double* u = Ux + (long long)e * (J + 2) * L1 + r;
    DU[t] = u[L1] - u[0];
  }
}

void wr_diff_u(int E, int nc, int d1, int J, const double* Ux_new, double* DU,
               cudaStream_t st) {
  long long L1 = (long long)d1 * nc;
  long long total = L1 * J * E;
  if (total == 0) return;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  wr_diff_u_kernel<<<blocks, 256, 0, st>>>(L1, J, E, Ux_new, DU);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// Modal w recursion (setup_modal): z_{s+1} = lam z_s + h_s for every (member, mode i,
// interval n), in place over Z = H (J blocks of a d2 x nc column-major matrix), z_{-1} = Z0.
// One thread per (e, i, n); consecutive threads walk consecutive modes, so every block
// access is coalesced.  The loads of 8 steps are issued before their dependent FMAs.
constexpr int SCAN_DEPTH = 8;
__global__ void wr_modal_scan_kernel(long long L2, int d2, int J, int E,
                                     const double* __restrict__ lam,
                                     const double* __restrict__ Z0, double* __restrict__ Z) {
  const long long total = L2 * E;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / L2);
    const long long r = t - e * L2;
    const double l = lam[(long long)e * d2 + (int)(r % d2)];
    double z = Z0[t];
    double* p = Z + (long long)e * J * L2 + r;
    int s = 0;
    for (; s + SCAN_DEPTH <= J; s += SCAN_DEPTH) {
      double h[SCAN_DEPTH];
#pragma unroll
      for (int q = 0; q < SCAN_DEPTH; ++q) h[q] = p[(long long)(s + q) * L2];
#pragma unroll
      for (int q = 0; q < SCAN_DEPTH; ++q) {
        z = fma(l, z, h[q]);
        p[(long long)(s + q) * L2] = z;
      }
    }
    for (; s < J; ++s) {
      z = fma(l, z, p[(long long)s * L2]);
      p[(long long)s * L2] = z;
    }
  }
}

void wr_modal_scan(int E, int nc, int d2, int J, const double* lam, const double* Z0, double* Z,
                   cudaStream_t st) {
  const long long L2 = (long long)d2 * nc;
  const long long total = L2 * E;
  if (total == 0 || J == 0) return;
  int blocks = (int)std::min<long long>((total + 127) / 128, 148 * 16);
  wr_modal_scan_kernel<<<blocks, 128, 0, st>>>(L2, d2, J, E, lam, Z0, Z);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// Deterministic warp sum: lane-strided partial sums then a fixed xor tree.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int COMMIT_THREADS = 256;
constexpr int COMMIT_WARPS = COMMIT_THREADS / 32;

// One warp per (interval, substep) row: ||dU_s||, ||dW_s|| into nrm[en][s][2], commit
// new -> cur (allatonce.py:256) and DW for the next rhs.
__device__ __forceinline__ void wr_commit_rows(int en, int s, int lane, int nc, int d1, int d2,
                                               int J, double* Ux_cur, const double* __restrict__ Ux_new,
                                               double* Wx_cur, const double* __restrict__ Wx_new,
                                               double* nrm, double* DW) {
  const int e = en / nc, n = en - (en / nc) * nc;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const long long bu = (long long)e * (J + 2) * L1 + (long long)(s + 2) * L1 + (long long)n * d1;
  const long long bw = (long long)e * (J + 2) * L2 + (long long)(s + 2) * L2 + (long long)n * d2;
  // Each lane keeps the lane-strided element order (i = lane + 32 c) of the summation but
  // issues all loads of a chunk before using them (memory-level parallelism; the row is
  // ~300 doubles, one chunk).
  constexpr int CPL = 10;
  double a = 0.0, b = 0.0;
  for (int base = 0; base < d1; base += 32 * CPL) {
    double vn[CPL], vc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = base + c * 32 + lane;
      if (i < d1) {
        vn[c] = Ux_new[bu + i];
        vc[c] = Ux_cur[bu + i];
      }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = base + c * 32 + lane;
      if (i < d1) {
        const double x = vn[c] - vc[c];
        a += x * x;
        Ux_cur[bu + i] = vn[c];
      }
    }
  }
  // DW_{s+1} = W_s - W_{s-1} for the next sweep's build_rhs (DW_0 = 0 stays from init)
  double* dw = (DW && s + 1 < J)
                   ? DW + (long long)e * J * L2 + (long long)(s + 1) * L2 + (long long)n * d2
                   : nullptr;
  for (int base = 0; base < d2; base += 32 * CPL) {
    double vn[CPL], vc[CPL], vp[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = base + c * 32 + lane;
      if (i < d2) {
        vn[c] = Wx_new[bw + i];
        vc[c] = Wx_cur[bw + i];
        if (dw) vp[c] = Wx_new[bw - L2 + i];
      }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = base + c * 32 + lane;
      if (i < d2) {
        const double x = vn[c] - vc[c];
        b += x * x;
        Wx_cur[bw + i] = vn[c];
        if (dw) dw[i] = vn[c] - vp[c];
      }
    }
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    nrm[((long long)en * J + s) * 2] = sqrt(a);
    nrm[((long long)en * J + s) * 2 + 1] = sqrt(b);
  }
}

// Stop decision for one interval, one warp: residual = max_s ||dU_s|| + max_s ||dW_s||
// (:250-254), u_final_prev update (:257), stop tests tol / diverged / floor (:258-271)
// and the max_iter cap.  nrm was written by other CTAs of the same launch: read from L2.
__device__ void wr_decide_interval(int en, int lane, int nc, int d1, int d2, int J, double alpha,
                                   double tol, int max_iter, const double* __restrict__ Ux_new,
                                   double* V, WrColumnState* cs, const double* nrm,
                                   double* resid_hist, int* active_count) {
  double mu = 0.0, mw = 0.0;
  for (int s = lane; s < J; s += 32) {
    const double a = __ldcg(nrm + ((long long)en * J + s) * 2);
    const double b = __ldcg(nrm + ((long long)en * J + s) * 2 + 1);
    mu = (a > mu || a != a) ? a : mu;
    mw = (b > mw || b != b) ? b : mw;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a = __shfl_xor_sync(0xffffffffu, mu, o), b = __shfl_xor_sync(0xffffffffu, mw, o);
    mu = (a > mu || a != a) ? a : mu;
    mw = (b > mw || b != b) ? b : mw;
  }
  if (d1 > 0) {  // V = u_start - alpha * u_final_prev with the new last row
    const int e = en / nc, n = en - (en / nc) * nc;
    const long long L1 = (long long)d1 * nc;
    const double* un = Ux_new + (long long)e * (J + 2) * L1 + (long long)n * d1;
    double* v = V + (long long)e * L1 + (long long)n * d1;
    const long long last = (long long)(J + 1) * L1;
    for (int i = lane; i < d1; i += 32) v[i] = un[i] - alpha * un[last + i];
  }
  if (lane == 0) {
    double resid = 0.0;
    if (d1 > 0) resid += mu;
    if (d2 > 0) resid += mw;
    WrColumnState c = cs[en];
    const bool go = wr_stop_update(c, resid, tol, max_iter,
                                   resid_hist ? resid_hist + (long long)en * max_iter : nullptr);
    cs[en] = c;
    if (go) atomicAdd(active_count, 1);
  }
}

// One CTA per (member, interval, 8 substeps): the rows, then (last CTA) the decision.
// Phase 1 (wide): one warp per (member, interval, substep) row: ||dU_s||, ||dW_s|| into
// nrm[en][s][2] and, for intervals still iterating, commit new -> cur (allatonce.py:256).
__global__ void __launch_bounds__(COMMIT_THREADS)
    wr_commit_norms_kernel(int nc, int d1, int d2, int J, double* Ux_cur,
                           const double* __restrict__ Ux_new, double* Wx_cur,
                           const double* __restrict__ Wx_new, WrColumnState* cs,
                           double* nrm, double* DW, double alpha, double tol, int max_iter,
                           double* V, double* resid_hist, int* active_count,
                           unsigned* ticket) {
  const int en = blockIdx.x;
  const int s = blockIdx.y * COMMIT_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (!cs[en].active) return;  // block-uniform
  if (s < J) wr_commit_rows(en, s, lane, nc, d1, d2, J, Ux_cur, Ux_new, Wx_cur, Wx_new, nrm, DW);
  // the last CTA of this interval (ticket) runs the stop decision: no second launch
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = (atomicAdd(ticket + en, 1u) == gridDim.y - 1);
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) ticket[en] = 0u;  // self-resetting for the next sweep
  __threadfence();
  if ((threadIdx.x >> 5) == 0)
    wr_decide_interval(en, lane, nc, d1, d2, J, alpha, tol, max_iter, Ux_new, V, cs, nrm,
                       resid_hist, active_count);
}

void wr_commit(int E, int nc, int d1, int d2, int J, double alpha, double tol, int max_iter,
               int /*sweep*/, double* Ux_cur, const double* Ux_new, double* Wx_cur,
               const double* Wx_new, double* V, WrColumnState* cs, double* resid_hist,
               int* active_count, double* nrm, double* DW, unsigned* ticket, cudaStream_t st) {
  dim3 g1(E * nc, (J + COMMIT_WARPS - 1) / COMMIT_WARPS);
  wr_commit_norms_kernel<<<g1, COMMIT_THREADS, 0, st>>>(nc, d1, d2, J, Ux_cur, Ux_new, Wx_cur,
                                                        Wx_new, cs, nrm, DW, alpha, tol,
                                                        max_iter, V, resid_hist, active_count,
                                                        ticket);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// Final state of each interval = last rows of the committed waveforms (:280-289).
__global__ void wr_finish_kernel(int E, int nc, int d1, int d2, int J,
                                 const double* __restrict__ Ux, const double* __restrict__ Wx,
                                 const WrColumnState* __restrict__ cs, double* X_out,
                                 int* sweeps, int* reasons) {
  const int d = d1 + d2;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const long long total = (long long)E * nc * d;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t % d);
    const long long en = t / d;
    const int n = (int)(en % nc), e = (int)(en / nc);
    double v;
    if (r < d1)
      v = Ux[(long long)e * (J + 2) * L1 + (long long)(J + 1) * L1 + (long long)n * d1 + r];
    else
      v = Wx[(long long)e * (J + 2) * L2 + (long long)(J + 1) * L2 + (long long)n * d2 + (r - d1)];
    X_out[t] = v;
    if (r == 0) {
      if (sweeps) sweeps[en] = cs[en].iterations;
      if (reasons) reasons[en] = cs[en].reason;
    }
  }
}

void wr_finish(int E, int nc, int d1, int d2, int J, const double* Ux_cur, const double* Wx_cur,
               const WrColumnState* cs, double* X_out, int* sweeps, int* reasons,
               cudaStream_t st) {
  long long total = (long long)E * nc * (d1 + d2);
  int blocks = (int)std::min<long long>((total + 255) / 256 + 1, 148 * 8);
  wr_finish_kernel<<<blocks, 256, 0, st>>>(E, nc, d1, d2, J, Ux_cur, Wx_cur, cs, X_out, sweeps,
                                           reasons);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// out[e][n][b][i] = X[e][b+1][n*dd + i], b = 0..J  (trajectory rows, allatonce.py:280-282)
__global__ void wr_gather_kernel(int E, int nc, int dd, int J, const double* __restrict__ X,
                                 double* __restrict__ out) {
  const long long L = (long long)dd * nc;
  const long long total = (long long)E * nc * (J + 1) * dd;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % dd);
    long long r = t / dd;
    const int b = (int)(r % (J + 1));
    r /= (J + 1);
    const int n = (int)(r % nc), e = (int)(r / nc);
    out[t] = X[(long long)e * (J + 2) * L + (long long)(b + 1) * L + (long long)n * dd + i];
  }
}

void wr_gather(int E, int nc, int dd, int J, const double* X, double* out, cudaStream_t st) {
  long long total = (long long)E * nc * (J + 1) * dd;
  if (total == 0) return;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  wr_gather_kernel<<<blocks, 256, 0, st>>>(E, nc, dd, J, X, out);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

__global__ void sub_kernel(long long n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    out[t] = a[t] - b[t];
}

void sub(long long n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n == 0) return;
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  sub_kernel<<<blocks, 256, 0, st>>>(n, a, b, out);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe
