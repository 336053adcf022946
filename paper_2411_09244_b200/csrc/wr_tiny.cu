// Fused waveform relaxation for small reduced systems (latency regime: BASELINE configs
// 0/1, d1, d2 <= ~64): one CTA per (member, interval) runs the WHOLE WR solve
// (allatonce.py:232-298) in one launch -- build_rhs, the alpha-circulant transforms (half
// spectrum, same pseudo-mode packing as the large path), the shifted complex solves, the
// w-sweep recursion, the residual and the reference's stop logic -- looping over sweeps
// on the device until this interval stops.  The interval's waveforms live in shared
// memory with the small operators (transposed, k-major); the shifted-solve blocks Bk too
// when they fit (cfg1: 160 KB), else they stream through L1/L2 with coalesced reads.  Every phase has a
// fixed per-output summation order (deterministic, batch invariant: each interval is
// computed by identical code in its own CTA).

#include <algorithm>
#include <cmath>

#include "pe.h"
#include "pe_internal.h"

namespace pe {

constexpr int TINY_MAX_THREADS = 512;

struct TinyArgs {
  int d1, d2, J, npm, nc, max_iter, bk_smem;
  double alpha, tol;
  // operators, per-member strides
  const double *RW, *M11dt, *Finv, *Fw, *GW, *cg, *Emat, *f1;
  long long s_rw, s_m11, s_bk, s_gw, s_cg, s_e, s_f1;
  const double* BkT;   // per pseudo-mode transposed blocks: [m][j][row], coalesced reads
  const double* X_in;  // (E, nc, d)
  double* X_out;
  int* sweeps;
  int* reasons;
  double* resid_hist;        // (E, nc, max_iter)
  double *Ux_cur, *Wx_cur;   // large-path waveform layout, filled at the end (readback)
};

__device__ __forceinline__ double tiny_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_k a[k sa] b[k sb] with four interleaved accumulators (fixed order: deterministic)
__device__ __forceinline__ double tdot(const double* a, int sa, const double* b, int sb, int n) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int k = 0;
#pragma unroll 2
  for (; k + 4 <= n; k += 4) {
    c0 = fma(a[(long long)k * sa], b[k * sb], c0);
    c1 = fma(a[(long long)(k + 1) * sa], b[(k + 1) * sb], c1);
    c2 = fma(a[(long long)(k + 2) * sa], b[(k + 2) * sb], c2);
    c3 = fma(a[(long long)(k + 3) * sa], b[(k + 3) * sb], c3);
  }
  for (; k < n; ++k) c0 = fma(a[(long long)k * sa], b[k * sb], c0);
  return (c0 + c1) + (c2 + c3);
}

// sum_k a[k sa] (b[k] - bp[k]) (difference-first lag, same as the large path's [X; DX])
__device__ __forceinline__ double tdotd(const double* a, int sa, const double* b, const double* bp,
                                        int n) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int k = 0;
#pragma unroll 2
  for (; k + 4 <= n; k += 4) {
    c0 = fma(a[(long long)k * sa], b[k] - bp[k], c0);
    c1 = fma(a[(long long)(k + 1) * sa], b[k + 1] - bp[k + 1], c1);
    c2 = fma(a[(long long)(k + 2) * sa], b[k + 2] - bp[k + 2], c2);
    c3 = fma(a[(long long)(k + 3) * sa], b[k + 3] - bp[k + 3], c3);
  }
  for (; k < n; ++k) c0 = fma(a[(long long)k * sa], b[k] - bp[k], c0);
  return (c0 + c1) + (c2 + c3);
}

__global__ void __launch_bounds__(TINY_MAX_THREADS) wr_tiny_kernel(const __grid_constant__ TinyArgs a) {
  const int en = blockIdx.x;
  const int e = en / a.nc, n = en - (en / a.nc) * a.nc;
  const int d1 = a.d1, d2 = a.d2, J = a.J, R2 = 2 * a.npm, d = d1 + d2;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int NW = nt >> 5;
  extern __shared__ double sm[];
  // rows 0..J: row 0 = interval start, row s+1 = waveform at substep s
  double* Uc = sm;                       // (J+1) x d1 committed
  double* Un = Uc + (J + 1) * d1;        // (J+1) x d1 candidate
  double* Wc = Un + (J + 1) * d1;        // (J+1) x d2
  double* Wn = Wc + (J + 1) * d2;        // (J+1) x d2
  double* R = Wn + (J + 1) * d2;         // J x d1
  double* P = R + J * d1;                // R2 x d1
  double* Q = P + R2 * d1;               // R2 x d1
  double* G = Q + R2 * d1;               // J x d2
  double* V = G + J * d2;                // d1
  double* nrm = V + d1;                  // 2 x J
  // small operators staged once, transposed (k-major): consecutive threads (rows i) read
  // consecutive words -> conflict-free
  double* RWT = nrm + 2 * J;             // 2 d2 x d1
  double* GWT = RWT + 2 * d2 * d1;       // 2 d1 x d2
  double* ET = GWT + 2 * d1 * d2;        // d2 x d2
  double* FiS = ET + d2 * d2;            // R2 x J   forward transform rows
  double* FwS = FiS + R2 * J;            // J x R2   backward transform rows
  double* BkS = FwS + J * R2;            // npm x 2d1 x 2d1 (transposed), when a.bk_smem
  __shared__ int s_stop, s_it, s_stall, s_reason;
  __shared__ double s_prev, s_r0;

  const double* RW = a.RW + e * a.s_rw;
  const double* M11dt = a.M11dt + e * a.s_m11;
  const double* GW = a.GW + e * a.s_gw;
  const double* cg = a.cg + e * a.s_cg;
  const double* Em = a.Emat + e * a.s_e;
  const double* f1 = a.f1 + e * a.s_f1;
  const double* x0 = a.X_in + (long long)en * d;

  for (int t = tid; t < d1 * 2 * d2; t += nt) {
    const int i = t / (2 * d2), k = t - (t / (2 * d2)) * 2 * d2;
    RWT[k * d1 + i] = __ldg(RW + t);
  }
  for (int t = tid; t < d2 * 2 * d1; t += nt) {
    const int q = t / (2 * d1), k = t - (t / (2 * d1)) * 2 * d1;
    GWT[k * d2 + q] = __ldg(GW + t);
  }
  for (int t = tid; t < d2 * d2; t += nt) ET[(t % d2) * d2 + t / d2] = __ldg(Em + t);
  for (int t = tid; t < R2 * J; t += nt) {
    FiS[t] = __ldg(a.Finv + t);
    FwS[t] = __ldg(a.Fw + t);
  }
  const double* Bk = a.BkT + e * a.s_bk;
  if (a.bk_smem) {
    for (long long t = tid; t < a.s_bk; t += nt) BkS[t] = __ldg(Bk + t);
    Bk = BkS;
  }
  // seeds (:239-241): U = u0, W = w0 on every row; u_final_prev = u0
  for (int t = tid; t < (J + 1) * d1; t += nt) {
    const double v = x0[t % d1];
    Uc[t] = v;
    Un[t] = v;
  }
  for (int t = tid; t < (J + 1) * d2; t += nt) {
    const double v = x0[d1 + t % d2];
    Wc[t] = v;
    Wn[t] = v;
  }
  for (int i = tid; i < d1; i += nt) V[i] = x0[i] - a.alpha * x0[i];
  if (tid == 0) {
    s_stop = 0;
    s_it = 0;
    s_stall = 0;
    s_reason = PE_STOP_MAX_ITER;
    s_prev = INFINITY;
    s_r0 = 0.0;
  }
  double* rh = a.resid_hist ? a.resid_hist + (long long)en * a.max_iter : nullptr;
  if (rh)
    for (int t = tid; t < a.max_iter; t += nt) rh[t] = NAN;
  __syncthreads();

  while (true) {
    if (d1 > 0) {
      // build_rhs (:136-158): R_s = f1 - A12 w_{s} - M12 (w_s - w_{s-1})/dt, w_s = Wc[s]
      for (int t = tid; t < J * d1; t += nt) {
        const int s = t / d1, i = t - (t / d1) * d1;
        double acc = tdot(RWT + i, d1, Wc + s * d2, 1, d2);
        if (s > 0) acc += tdotd(RWT + d2 * d1 + i, d1, Wc + s * d2, Wc + (s - 1) * d2, d2);
        double v = acc + __ldg(f1 + i);
        if (s == 0) v = v + tdot(M11dt + (long long)i * d1, 1, V, 1, d1);  // + M11 v / dt
        R[t] = v;
      }
      __syncthreads();
      // P = S^{-1} R (half spectrum, pseudo-mode planes)
      for (int t = tid; t < R2 * d1; t += nt) {
        const int r = t / d1, i = t - (t / d1) * d1;
        P[t] = tdot(FiS + r * J, 1, R + i, d1, J);
      }
      __syncthreads();
      // Q_m = Bk_m P_m (shifted complex inverses as real 2x2-block matrices)
      for (int t = tid; t < R2 * d1; t += nt) {
        const int r = t / d1, i = t - (t / d1) * d1;
        const int m = r >> 1, a2 = r & 1;
        Q[t] = tdot(Bk + (long long)m * 4 * d1 * d1 + a2 * d1 + i, 2 * d1, P + m * 2 * d1, 1,
                    2 * d1);
      }
      __syncthreads();
      // U = Re(S Q): candidate rows 1..J
      for (int t = tid; t < J * d1; t += nt) {
        const int s = t / d1, i = t - (t / d1) * d1;
        Un[(s + 1) * d1 + i] = tdot(FwS + s * R2, 1, Q + i, d1, R2);
      }
      __syncthreads();
    }
    if (d2 > 0) {
      // g_s = cg + Gu U_s + Gd (U_{s-1} - U_{s-2})  (_w_sweep :222-224)
      for (int t = tid; t < J * d2; t += nt) {
        const int s = t / d2, q = t - (t / d2) * d2;
        double acc = tdot(GWT + q, d2, Un + (s + 1) * d1, 1, d1);
        if (s > 0) acc += tdotd(GWT + d1 * d2 + q, d2, Un + s * d1, Un + (s - 1) * d1, d1);
        G[t] = acc + __ldg(cg + q);
      }
      __syncthreads();
      // w_{s+1} = E w_s + g_s, sequential in s (:226-229): one warp, warp-level ordering
      if (warp == 0) {
        for (int s = 0; s < J; ++s) {
          for (int q = lane; q < d2; q += 32)
            Wn[(s + 1) * d2 + q] = tdot(ET + q, d2, Wn + s * d2, 1, d2) + G[s * d2 + q];
          __syncwarp();
        }
      }
      __syncthreads();
    }
    // residual = max_s ||dU_s|| + max_s ||dW_s|| (:250-254); warp per substep
    for (int s = warp; s < J; s += NW) {
      double x = 0.0, y = 0.0;
      for (int i = lane; i < d1; i += 32) {
        const double df = Un[(s + 1) * d1 + i] - Uc[(s + 1) * d1 + i];
        x += df * df;
      }
      for (int i = lane; i < d2; i += 32) {
        const double df = Wn[(s + 1) * d2 + i] - Wc[(s + 1) * d2 + i];
        y += df * df;
      }
      x = tiny_warp_sum(x);
      y = tiny_warp_sum(y);
      if (lane == 0) {
        nrm[s] = sqrt(x);
        nrm[J + s] = sqrt(y);
      }
    }
    __syncthreads();
    // commit (:256) and u_final_prev (:257)
    for (int t = tid + d1; t < (J + 1) * d1; t += nt) Uc[t] = Un[t];
    for (int t = tid + d2; t < (J + 1) * d2; t += nt) Wc[t] = Wn[t];
    if (tid == 0) {
      double mu = 0.0, mw = 0.0;
      for (int s = 0; s < J; ++s) {
        mu = (nrm[s] > mu || nrm[s] != nrm[s]) ? nrm[s] : mu;
        mw = (nrm[J + s] > mw || nrm[J + s] != nrm[J + s]) ? nrm[J + s] : mw;
      }
      double resid = 0.0;
      if (d1 > 0) resid += mu;
      if (d2 > 0) resid += mw;
      const int it = s_it;
      if (rh) rh[it] = resid;
      if (it == 0) s_r0 = resid;
      s_it = it + 1;
      int stop = 0;
      if (resid <= a.tol) {
        s_reason = PE_STOP_TOL;
        stop = 1;
      } else if (!isfinite(resid) || resid > 1e8 * fmax(1.0, s_r0)) {
        s_reason = PE_STOP_DIVERGED;
        stop = 1;
      } else {
        s_stall = (resid >= s_prev) ? s_stall + 1 : 0;
        if (s_stall >= 2 && resid <= 1e3 * a.tol) {
          s_reason = PE_STOP_FLOOR;
          stop = 1;
        }
        s_prev = resid;
      }
      if (!stop && s_it >= a.max_iter) {
        s_reason = PE_STOP_MAX_ITER;
        stop = 1;
      }
      s_stop = stop;
    }
    __syncthreads();
    for (int i = tid; i < d1; i += nt) V[i] = Uc[i] - a.alpha * Uc[J * d1 + i];
    if (s_stop) break;
    __syncthreads();
  }
  // outputs: final state = last rows (:280-289); waveforms in the large-path layout
  double* xo = a.X_out + (long long)en * d;
  for (int i = tid; i < d1; i += nt) xo[i] = Uc[J * d1 + i];
  for (int i = tid; i < d2; i += nt) xo[d1 + i] = Wc[J * d2 + i];
  const long long L1 = (long long)d1 * a.nc, L2 = (long long)d2 * a.nc;
  for (int t = tid; t < (J + 1) * d1; t += nt) {
    const int b = t / d1, i = t - (t / d1) * d1;
    a.Ux_cur[(long long)e * (J + 2) * L1 + (long long)(b + 1) * L1 + (long long)n * d1 + i] = Uc[t];
  }
  for (int t = tid; t < (J + 1) * d2; t += nt) {
    const int b = t / d2, i = t - (t / d2) * d2;
    a.Wx_cur[(long long)e * (J + 2) * L2 + (long long)(b + 1) * L2 + (long long)n * d2 + i] = Wc[t];
  }
  if (tid == 0) {
    if (a.sweeps) a.sweeps[en] = s_it;
    if (a.reasons) a.reasons[en] = s_reason;
  }
}

size_t wr_tiny_smem(int d1, int d2, int J, int npm) {
  return sizeof(double) * ((size_t)2 * (J + 1) * d1 + 2 * (size_t)(J + 1) * d2 + (size_t)J * d1 +
                           4 * (size_t)npm * d1 + (size_t)J * d2 + d1 + 2 * (size_t)J +
                           4 * (size_t)d1 * d2 + (size_t)d2 * d2 + 4 * (size_t)npm * J);
}

static size_t tiny_bk_bytes(int d1, int npm) { return sizeof(double) * 4 * (size_t)npm * d1 * d1; }
static constexpr size_t TINY_SMEM_CAP = 225 * 1024;  // below the 227 KB opt-in limit

// Fused path when the per-interval working set fits in shared memory and the operators
// are small (latency regime).
bool wr_tiny_eligible(int d1, int d2, int J, int npm) {
  return d1 <= 96 && d2 <= 96 && J <= 128 && wr_tiny_smem(d1, d2, J, npm) <= 160 * 1024;
}

void wr_tiny(const TinyArgsPublic& p, cudaStream_t st) {
  TinyArgs a;
  a.d1 = p.d1;
  a.d2 = p.d2;
  a.J = p.J;
  a.npm = p.npm;
  a.nc = p.nc;
  a.max_iter = p.max_iter;
  a.alpha = p.alpha;
  a.tol = p.tol;
  a.RW = p.RW;
  a.M11dt = p.M11dt;
  a.Finv = p.Finv;
  a.Fw = p.Fw;
  a.GW = p.GW;
  a.cg = p.cg;
  a.Emat = p.Emat;
  a.f1 = p.f1;
  a.BkT = p.BkT;
  a.s_rw = 2LL * p.d1 * p.d2;
  a.s_m11 = (long long)p.d1 * p.d1;
  a.s_bk = (long long)p.npm * 4 * p.d1 * p.d1;
  a.s_gw = 2LL * p.d1 * p.d2;
  a.s_cg = p.d2;
  a.s_e = (long long)p.d2 * p.d2;
  a.s_f1 = p.d1;
  a.X_in = p.X_in;
  a.X_out = p.X_out;
  a.sweeps = p.sweeps;
  a.reasons = p.reasons;
  a.resid_hist = p.resid_hist;
  a.Ux_cur = p.Ux_cur;
  a.Wx_cur = p.Wx_cur;
  size_t smem = wr_tiny_smem(p.d1, p.d2, p.J, p.npm);
  a.bk_smem = smem + tiny_bk_bytes(p.d1, p.npm) <= TINY_SMEM_CAP;
  if (a.bk_smem) smem += tiny_bk_bytes(p.d1, p.npm);
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(wr_tiny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)TINY_SMEM_CAP));
    attr = true;
  }
  // one thread per output of the widest phase (J d1, 2 npm d1, J d2), whole warps
  int work = std::max(p.J * p.d1, std::max(2 * p.npm * p.d1, p.J * p.d2));
  int nt = std::min(TINY_MAX_THREADS, std::max(128, (work + 31) / 32 * 32));
  wr_tiny_kernel<<<p.E * p.nc, nt, smem, st>>>(a);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe
