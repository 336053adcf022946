// Reference-API building blocks of the all-at-once solver and the initial projection,
// exported for drop-in callers (the hot path fuses these into the WR sweep):
//
//   pe_apply_S          apply_S / apply_S_inverse        allatonce.py:74-88
//   pe_build_rhs        build_rhs                        allatonce.py:136-158
//   pe_allatonce_usolve ImplicitAllAtOnce.solve          allatonce.py:112-133
//   pe_project_initial  project_initial                  stepping.py:216-226
//
// All arithmetic in FP64 with fixed reduction orders (deterministic).

#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "pe.h"
#include "pe_ctx.h"

namespace pe {

extern long long g_launches;

namespace {

// ------------------------------------------------------------------ S and S^-1
// x, y: (J, ncols) row-major (time on axis 0, as numpy's axis-0 FFTs); planar re / im.
//   inverse: y_t = (1/J) sum_s e^{-2 pi i t s / J} alpha^{s/J} x_s     (fft(x / Lambda) / J)
//   forward: y_t = alpha^{-t/J} sum_s e^{+2 pi i t s / J} x_s          (Lambda J ifft(x))
// Direct DFT, s ascending; the twiddle angle is reduced exactly ((t s) mod J) first.
__global__ void k_apply_S(int J, long long ncols, double alpha, int inverse,
                          const double* __restrict__ xr, const double* __restrict__ xi,
                          double* __restrict__ yr, double* __restrict__ yi) {
  const long long total = (long long)J * ncols;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(q / ncols);
    const long long c = q - (long long)t * ncols;
    double ar = 0.0, ai = 0.0;
    for (int s = 0; s < J; ++s) {
      const long long m = ((long long)t * s) % J;
      double sn, cs;
      sincospi(2.0 * (double)m / (double)J, &sn, &cs);
      if (inverse) sn = -sn;
      double vr = xr[(long long)s * ncols + c];
      double vi = xi ? xi[(long long)s * ncols + c] : 0.0;
      if (inverse) {
        const double w = pow(alpha, (double)s / (double)J);
        vr *= w;
        vi *= w;
      }
      ar = fma(cs, vr, fma(-sn, vi, ar));
      ai = fma(cs, vi, fma(sn, vr, ai));
    }
    if (inverse) {
      ar /= J;
      ai /= J;
    } else {
      const double l = pow(alpha, -(double)t / (double)J);
      ar *= l;
      ai *= l;
    }
    yr[q] = ar;
    if (yi) yi[q] = ai;
  }
}

// ------------------------------------------------------------------ build_rhs
// One warp per (s, i): rhs_s = f1_s - M12 (wh_{s+1} - wh_s) / dt - A12 wh_{s+1}
// (+ M11 (u_start - alpha u_final_prev) / dt on row 0), wh = [w_lag, w_start, W_prev[:-1]].
__device__ __forceinline__ const double* wh_row(int r, const double* w_lag, const double* w_start,
                                                const double* Wp, int d2) {
  return r == 0 ? w_lag : (r == 1 ? w_start : Wp + (long long)(r - 2) * d2);
}

__global__ void k_build_rhs(int d1, int d2, int J, const double* __restrict__ M11,
                            const double* __restrict__ M12, const double* __restrict__ A12,
                            const double* __restrict__ f1, const double* __restrict__ u_start,
                            const double* __restrict__ w_start, const double* __restrict__ w_lag,
                            const double* __restrict__ Wp, const double* __restrict__ ufp,
                            double dt, double alpha, double* __restrict__ rhs) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= (long long)J * d1) return;
  const int s = (int)(warp / d1), i = (int)(warp - (long long)s * d1);
  const double* a = wh_row(s, w_lag, w_start, Wp, d2);
  const double* b = wh_row(s + 1, w_lag, w_start, Wp, d2);
  double sm = 0.0, sa = 0.0, s0 = 0.0;
  for (int j = lane; j < d2; j += 32) {
    sm = fma(M12[(long long)i * d2 + j], (b[j] - a[j]) / dt, sm);
    sa = fma(A12[(long long)i * d2 + j], b[j], sa);
  }
  if (s == 0)
    for (int j = lane; j < d1; j += 32)
      s0 = fma(M11[(long long)i * d1 + j], u_start[j] - alpha * ufp[j], s0);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
  }
  if (lane == 0) {
    double r = f1[(long long)s * d1 + i] - sm - sa;
    if (s == 0) r += s0 / dt;
    rhs[(long long)s * d1 + i] = r;
  }
}

// ------------------------------------------------------------------ u solve helpers
// flat (E, nc, J, d1) <-> blocked (per member: J blocks of [n][i], block s at blk_off +
// s nc d1, member stride blk_es).  to_blocks: blocked <- flat, else flat <- blocked.
__global__ void k_permute_nsi(long long E, int nc, int J, int d1, double* flat, double* blocked,
                              long long blk_es, long long blk_off, int to_blocks) {
  const long long per = (long long)nc * J * d1, total = E * per;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / per;
    long long r = q - e * per;
    const int n = (int)(r / ((long long)J * d1));
    r -= (long long)n * J * d1;
    const int s = (int)(r / d1), i = (int)(r - (long long)s * d1);
    const long long blk = blk_off + e * blk_es + ((long long)s * nc + n) * d1 + i;
    if (to_blocks)
      blocked[blk] = flat[q];
    else
      flat[q] = blocked[blk];
  }
}

// modal coordinates, layout [e][n][s][i]: (B + mu_i) y_i = r_i per (e, n, i), the
// alpha-circulant bidiagonal B closed at its corner (wr_modal.cu, modal_uscan_kernel)
__global__ void k_modal_usolve(long long E, int nc, int d1, int J, double dt, double alpha,
                               const double* __restrict__ acoef, const double* __restrict__ cden,
                               const double* __restrict__ Rt, double* __restrict__ Y) {
  const long long total = E * nc * d1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / ((long long)nc * d1);
    const long long r = q - e * nc * d1;
    const int n = (int)(r / d1), i = (int)(r - (long long)n * d1);
    const double a = acoef[e * d1 + i], cd = cden[e * d1 + i];
    const double* rp = Rt + (e * nc + n) * (long long)J * d1 + i;
    double* yp = Y + (e * nc + n) * (long long)J * d1 + i;
    double c = 0.0;
    for (int s = 1; s < J; ++s) c = a * fma(dt, rp[(long long)s * d1], c);
    double y = a * fma(alpha, c, dt * rp[0]) * cd;
    yp[0] = y;
    for (int s = 1; s < J; ++s) {
      y = a * fma(dt, rp[(long long)s * d1], y);
      yp[(long long)s * d1] = y;
    }
  }
}

// residual of the stacked system, row form as ImplicitAllAtOnce.solve (allatonce.py:125-131):
// res_s = bu_s M11 + u_s A11 - rhs_s, bu_0 = (u_0 - alpha u_{J-1}) / dt, bu_s = (u_s - u_{s-1}) / dt.
// One CTA per (e, n, s): partial sums of |res|^2 and |rhs|^2 (fixed order).
__global__ void k_aao_residual(int nc, int d1, int J, double dt, double alpha,
                               const double* __restrict__ M11, const double* __restrict__ A11,
                               long long mstride, const double* __restrict__ U,
                               const double* __restrict__ R, double* __restrict__ part) {
  const int s = blockIdx.x, n = blockIdx.y, e = blockIdx.z;
  const double* u = U + ((long long)e * nc + n) * (long long)J * d1;
  const double* rh = R + ((long long)e * nc + n) * (long long)J * d1;
  const double* m = M11 + e * mstride;
  const double* a = A11 + e * mstride;
  const double* us = u + (long long)s * d1;
  const double* up = u + (long long)(s ? s - 1 : J - 1) * d1;
  const double w = s ? 1.0 : alpha;
  double rr = 0.0, bb = 0.0;
  for (int i = threadIdx.x; i < d1; i += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < d1; ++j)
      acc = fma((us[j] - w * up[j]) / dt, m[(long long)j * d1 + i],
                fma(us[j], a[(long long)j * d1 + i], acc));
    const double r = acc - rh[(long long)s * d1 + i];
    rr = fma(r, r, rr);
    bb = fma(rh[(long long)s * d1 + i], rh[(long long)s * d1 + i], bb);
  }
  __shared__ double sr[256], sb[256];
  sr[threadIdx.x] = rr;
  sb[threadIdx.x] = bb;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      sr[threadIdx.x] += sr[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const long long k = (((long long)e * nc + n) * J + s) * 2;
    part[k] = sr[0];
    part[k + 1] = sb[0];
  }
}

__global__ void k_aao_residual_sum(long long cols, int J, const double* __restrict__ part,
                                   double* __restrict__ out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double r = 0.0, b = 0.0;
  for (int s = 0; s < J; ++s) {
    r += part[(c * J + s) * 2];
    b += part[(c * J + s) * 2 + 1];
  }
  out[c] = sqrt(r) / fmax(sqrt(b), 1e-300);
}


// WR solver-residual diagnostic inputs from the final waveforms (blocks 1..J+1 of
// Ux_cur / Wx_cur, member stride (J+2) L): DWdt_s = (W_{s+1} - W_s) / dt with
// DWdt_0 = 0 (w_lag = w_start), V = u_start - alpha u_J
__global__ void k_wr_diag_prep(int E, int J, long long L1, long long L2, double dt, double alpha,
                               const double* __restrict__ U, const double* __restrict__ W,
                               double* __restrict__ DWdt, double* __restrict__ V) {
  const long long nw = (long long)E * J * L2, total = nw + (long long)E * L1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    if (q < nw) {
      const long long e = q / (J * L2);
      const long long r = q - e * J * L2;
      const int sidx = (int)(r / L2);
      const long long x = r - (long long)sidx * L2;
      const double* w = W + e * (J + 2) * L2 + x;
      DWdt[q] = sidx == 0 ? 0.0 : (w[(long long)(sidx + 1) * L2] - w[(long long)sidx * L2]) / dt;
    } else {
      const long long t = q - nw;
      const long long e = t / L1, x = t - e * L1;
      const double* u = U + e * (J + 2) * L1 + x;
      V[t] = u[L1] - alpha * u[(long long)(J + 1) * L1];
    }
  }
}

// ------------------------------------------------------------------ projection helpers
__global__ void k_csr_spmv(int n, const int* __restrict__ p, const int* __restrict__ ix,
                           const double* __restrict__ v, const double* __restrict__ x,
                           double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int t = p[i]; t < p[i + 1]; ++t) s = fma(v[t], x[ix[t]], s);
  y[i] = s;
}

__global__ void k_csc_tdot(int d, const int* __restrict__ cp, const int* __restrict__ ci,
                           const double* __restrict__ cv, const double* __restrict__ b,
                           double* __restrict__ f) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= d) return;
  double s = 0.0;
  for (int t = cp[j] + lane; t < cp[j + 1]; t += 32) s = fma(cv[t], b[ci[t]], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) f[j] = s;
}

// ------------------------------------------------------------------ stability bound
// Power iteration of stepping.py:191-207 on P = M22^-1 A22: z = P v / ||P v||,
// lam = (z^T A22 z) / (z^T M22 z), stop when |lam_new - lam| <= tol |lam_new|.  One warp per
// row for the three products, block partials summed in a fixed order by one thread; every
// kernel returns at once when st[0] (done) is set, so batches of iterations can be enqueued.
struct PowerState {
  double lam, lam_new;
  int done, iters;
};

__global__ void k_pw_gemv(int n, const double* __restrict__ P, const double* __restrict__ v,
                          double* __restrict__ y, double* __restrict__ part,
                          const PowerState* ps) {
  if (ps->done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double wp[8];
  double acc2 = 0.0;
  for (int r = blockIdx.x * 8 + warp; r < n; r += gridDim.x * 8) {
    double a = 0.0;
    for (int k = lane; k < n; k += 32) a = fma(P[(long long)r * n + k], v[k], a);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      y[r] = a;
      acc2 = fma(a, a, acc2);
    }
  }
  if (lane == 0) wp[warp] = acc2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += wp[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_pw_rq(int n, const double* __restrict__ A, const double* __restrict__ M,
                        const double* __restrict__ y, const double* __restrict__ ypart, int nb,
                        double* __restrict__ z, double* __restrict__ part, const PowerState* ps) {
  if (ps->done) return;
  // every block recomputes ||y|| from the same partials in the same order (identical bits)
  __shared__ double nrm;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nb; ++b) t += ypart[b];
    nrm = sqrt(t);
  }
  __syncthreads();
  const double inv = nrm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double wa[8], wm[8];
  double sa = 0.0, sm = 0.0;
  for (int r = blockIdx.x * 8 + warp; r < n; r += gridDim.x * 8) {
    double a = 0.0, m = 0.0;
    for (int k = lane; k < n; k += 32) {
      const double zk = y[k] / inv;
      a = fma(A[(long long)r * n + k], zk, a);
      m = fma(M[(long long)r * n + k], zk, m);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if (lane == 0) {
      const double zr = y[r] / inv;
      z[r] = zr;
      sa = fma(zr, a, sa);
      sm = fma(zr, m, sm);
    }
  }
  if (lane == 0) {
    wa[warp] = sa;
    wm[warp] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tm = 0.0;
    for (int w = 0; w < 8; ++w) {
      ta += wa[w];
      tm += wm[w];
    }
    part[2 * blockIdx.x] = ta;
    part[2 * blockIdx.x + 1] = tm;
  }
}

__global__ void k_pw_finish(int nb, const double* __restrict__ part, double tol, int max_iter,
                            PowerState* ps) {
  if (ps->done) return;
  double ta = 0.0, tm = 0.0;
  for (int b = 0; b < nb; ++b) {
    ta += part[2 * b];
    tm += part[2 * b + 1];
  }
  const double lam_new = ta / tm;
  const bool done = fabs(lam_new - ps->lam) <= tol * fabs(lam_new);
  ps->lam = lam_new;
  ps->iters += 1;
  if (done || ps->iters >= max_iter) ps->done = done ? 1 : 2;
}

int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 32));
}

template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) {
    if (n) {
      cudaError_t e = cudaMalloc(&p, n * sizeof(T));
      if (e != cudaSuccess)
        throw Error{PE_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
    }
  }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

template <class F>
int api_guard(const char* name, F&& f) {
  try {
    f();
    return PE_OK;
  } catch (const Error& e) {
    set_error(std::string(name) + ": " + e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(std::string(name) + ": " + e.what());
    return PE_ERR_CUDA;
  }
}

void require_arg(bool ok, const char* msg) {
  if (!ok) throw Error{PE_ERR_ARG, msg};
}

}  // namespace

// Shared with pe_api.cu: the all-at-once u solve on the context's factorisation.
void allatonce_usolve(pe_ctx* c, const double* R, double* U, int nc, double* resid,
                      cudaStream_t st) {
  const int d1 = c->d1, J = c->J, E = c->E;
  if (!c->wr_ready) throw Error{PE_ERR_STATE, "pe_prepare_allatonce has not been called"};
  const long long per = (long long)E * nc * J * d1;
  if (per == 0) return;
  const double dt = c->wr_dt, alpha = c->wr_alpha;
  const long long vstride = (long long)d1 * d1 + (long long)c->d2 * c->d2;
  if (c->wr_modal_full) {
    // r~ = V1^T R, (B + mu) y = r~ per mode, U = V1 Y   (V1^T M11 V1 = I, V1^T A11 V1 = diag mu)
    c->R.ensure(sizeof(double) * per + 8);
    c->P.ensure(sizeof(double) * per + 8);
    auto basis = [&](const double* A, bool trans, const double* B, double* C) {
      GemmParams p;
      p.M = d1;
      p.N = nc * J;
      p.nb1 = E;
      p.nseg = 1;
      p.seg[0].A = trans ? Operand{A, 1, d1, vstride, 0} : Operand{A, d1, 1, vstride, 0};
      p.seg[0].B = Operand{B, 1, d1, (long long)nc * J * d1, 0};
      p.seg[0].K = d1;
      p.C = C;
      p.c_i = 1;
      p.c_j = d1;
      p.c_b1 = (long long)nc * J * d1;
      gemm_f64(p, st);
    };
    basis(c->Vcat.d(), true, R, c->R.d());
    k_modal_usolve<<<grid_for((long long)E * nc * d1, 128), 128, 0, st>>>(
        E, nc, d1, J, dt, alpha, c->acoef.d(), c->cden.d(), c->R.d(), c->P.d());
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
    basis(c->Vcat.d(), false, c->P.d(), U);
  } else {
    // general path: S^-1 along time (half spectrum), shifted inverses, Re(S .)
    const long long L1 = (long long)d1 * nc;
    const int nk = c->wr_nk;
    c->R.ensure(sizeof(double) * E * J * L1 + 8);
    c->P.ensure(sizeof(double) * E * 2 * nk * L1 + 8);
    c->Q.ensure(sizeof(double) * E * 2 * nk * L1 + 8);
    c->Ux_new.ensure(sizeof(double) * E * (J + 2) * L1 + 8);
    k_permute_nsi<<<grid_for(per, 256), 256, 0, st>>>(E, nc, J, d1, const_cast<double*>(R),
                                                       c->R.d(), J * L1, 0, 1);
    ++g_launches;
    GemmParams tf;
    tf.M = 2 * nk;
    tf.N = (int)L1;
    tf.nb1 = E;
    tf.nseg = 1;
    tf.seg[0].A = Operand{c->Finv.d(), J, 1, 0, 0};
    tf.seg[0].B = Operand{c->R.d(), L1, 1, J * L1, 0};
    tf.seg[0].K = J;
    tf.C = c->P.d();
    tf.c_i = L1;
    tf.c_j = 1;
    tf.c_b1 = 2 * nk * L1;
    gemm_f64(tf, st);
    GemmParams sh;
    sh.M = d1;
    sh.N = nc;
    sh.nb1 = E * nk;
    sh.nb2 = 2;
    sh.nseg = 2;
    sh.seg[0].A = Operand{c->Bk.d(), 2LL * d1, 1, 4LL * d1 * d1, 2LL * d1 * d1};
    sh.seg[0].B = Operand{c->P.d(), 1, d1, 2 * L1, 0};
    sh.seg[0].K = d1;
    sh.seg[1].A = Operand{c->Bk.d() + d1, 2LL * d1, 1, 4LL * d1 * d1, 2LL * d1 * d1};
    sh.seg[1].B = Operand{c->P.d() + L1, 1, d1, 2 * L1, 0};
    sh.seg[1].K = d1;
    sh.C = c->Q.d();
    sh.c_i = 1;
    sh.c_j = d1;
    sh.c_b1 = 2 * L1;
    sh.c_b2 = L1;
    gemm_f64(sh, st);
    GemmParams tb;
    tb.M = J;
    tb.N = (int)L1;
    tb.nb1 = E;
    tb.nseg = 1;
    tb.seg[0].A = Operand{c->Fw.d(), 2LL * nk, 1, 0, 0};
    tb.seg[0].B = Operand{c->Q.d(), L1, 1, 2 * nk * L1, 0};
    tb.seg[0].K = 2 * nk;
    tb.C = c->Ux_new.d() + 2 * L1;
    tb.c_i = L1;
    tb.c_j = 1;
    tb.c_b1 = (J + 2) * L1;
    gemm_f64(tb, st);
    k_permute_nsi<<<grid_for(per, 256), 256, 0, st>>>(E, nc, J, d1, U, c->Ux_new.d(),
                                                       (J + 2) * L1, 2 * L1, 0);  // U <- blocks
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
  }
  if (resid) {
    Dev<double> part((size_t)E * nc * J * 2);
    dim3 g(J, nc, E);
    k_aao_residual<<<g, 256, 0, st>>>(nc, d1, J, dt, alpha, c->M11.d(), c->A11.d(),
                                       (long long)d1 * d1, U, R, part.p);
    k_aao_residual_sum<<<grid_for((long long)E * nc, 128), 128, 0, st>>>((long long)E * nc, J,
                                                                         part.p, resid);
    g_launches += 2;
    PE_CUDA_CHECK(cudaGetLastError());
    PE_CUDA_CHECK(cudaStreamSynchronize(st));  // `part` is freed on return
  }
}


// WRResult.solver_residual (allatonce.py:296): ImplicitAllAtOnce's conditioning guard
// (:125-131) for the intervals of the last all-at-once solve.  The rhs is build_rhs
// (:136-158) of each interval's final waveforms -- the system the sweep after the stop would
// solve; it differs from the last sweep's by at most the WR tolerance, which moves a
// relative residual of a linear solve only at rounding level -- solved on the context's
// factorisation, residual in the row form of :129-131.
void wr_solver_residual(pe_ctx* c, double* out, cudaStream_t st) {
  const int d1 = c->d1, d2 = c->d2, J = c->J, E = c->E, nc = c->wr_last_nc;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const double dt = c->wr_dt, alpha = c->wr_alpha;
  const double* U = c->Ux_cur.d();
  const double* W = c->Wx_cur.d();
  Dev<double> dw((size_t)E * J * L2 + 1), v((size_t)E * L1), rb((size_t)E * J * L1),
      rf((size_t)E * J * L1), uf((size_t)E * J * L1);
  k_wr_diag_prep<<<grid_for((long long)E * (J * L2 + L1), 256), 256, 0, st>>>(
      E, J, L1, L2, dt, alpha, U, W, dw.p, v.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  // R_s = f1_s - A12 wh_{s+1} - M12 (wh_{s+1} - wh_s) / dt, wh_{s+1} = W block s + 1
  GemmParams r;
  r.M = d1;
  r.N = J * nc;
  r.nb1 = E;
  r.alpha = -1.0;
  r.C = rb.p;
  r.c_i = 1;
  r.c_j = d1;
  r.c_b1 = J * L1;
  if (c->wr_last_loads) {
    r.Cin = c->LF1.d();  // [e][s][n][i]: the R block layout
    r.beta = 1.0;
  } else {
    r.bias = c->f1.d();
    r.bias_b1 = d1;
  }
  if (d2) {
    r.nseg = 2;
    r.seg[0].A = Operand{c->A12.d(), d2, 1, (long long)d1 * d2, 0};
    r.seg[0].B = Operand{W + L2, 1, d2, (J + 2) * L2, 0};
    r.seg[0].K = d2;
    r.seg[1].A = Operand{c->M12.d(), d2, 1, (long long)d1 * d2, 0};
    r.seg[1].B = Operand{dw.p, 1, d2, J * L2, 0};
    r.seg[1].K = d2;
    gemm_f64(r, st);
  } else {  // no w block: R = f1 rows
    r.nseg = 1;
    r.alpha = 0.0;
    r.seg[0].A = Operand{c->M11.d(), d1, 1, (long long)d1 * d1, 0};
    r.seg[0].B = Operand{U + L1, 1, d1, (J + 2) * L1, 0};
    r.seg[0].K = d1;
    gemm_f64(r, st);
  }
  // R_0 += M11 (u_start - alpha u_final) / dt
  GemmParams r0;
  r0.M = d1;
  r0.N = nc;
  r0.nb1 = E;
  r0.nseg = 1;
  r0.alpha = 1.0 / dt;
  r0.seg[0].A = Operand{c->M11.d(), d1, 1, (long long)d1 * d1, 0};
  r0.seg[0].B = Operand{v.p, 1, d1, L1, 0};
  r0.seg[0].K = d1;
  r0.C = rb.p;
  r0.c_i = 1;
  r0.c_j = d1;
  r0.c_b1 = J * L1;
  r0.Cin = rb.p;
  r0.beta = 1.0;
  gemm_f64(r0, st);
  const long long per = (long long)E * nc * J * d1;
  k_permute_nsi<<<grid_for(per, 256), 256, 0, st>>>(E, nc, J, d1, rf.p, rb.p, J * L1, 0, 0);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  allatonce_usolve(c, rf.p, uf.p, nc, out, st);  // synchronises before the buffers go
}
}  // namespace pe

using namespace pe;

extern "C" int pe_apply_S(int J, long long ncols, double alpha, int inverse, const double* xr,
                          const double* xi, double* yr, double* yi, void* stream) {
  return api_guard("pe_apply_S", [&] {
    require_arg(J >= 1 && ncols >= 0 && alpha > 0.0 && alpha < 1.0 && xr && yr,
                "need J >= 1, ncols >= 0, 0 < alpha < 1 and buffers");
    const long long total = (long long)J * ncols;
    if (!total) return;
    k_apply_S<<<grid_for(total, 128), 128, 0, (cudaStream_t)stream>>>(J, ncols, alpha, inverse,
                                                                      xr, xi, yr, yi);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
  });
}

extern "C" int pe_build_rhs(int d1, int d2, int J, const double* M11, const double* M12,
                            const double* A12, const double* f1_rows, const double* u_start,
                            const double* w_start, const double* w_lag,
                            const double* w_rows_prev, const double* u_final_prev, double dt,
                            double alpha, double* rhs, void* stream) {
  return api_guard("pe_build_rhs", [&] {
    require_arg(d1 >= 0 && d2 >= 0 && J >= 1 && dt > 0 && rhs && f1_rows,
                "need d1, d2 >= 0, J >= 1, dt > 0 and buffers");
    require_arg(d1 == 0 || (M11 && u_start && u_final_prev), "NULL u-block input");
    require_arg(d2 == 0 || d1 == 0 || (M12 && A12 && w_start && w_lag && w_rows_prev),
                "NULL w-block input");
    const long long warps = (long long)J * d1;
    if (!warps) return;
    k_build_rhs<<<grid_for(warps * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        d1, d2, J, M11, M12, A12, f1_rows, u_start, w_start, w_lag, w_rows_prev, u_final_prev,
        dt, alpha, rhs);
    ++g_launches;
    PE_CUDA_CHECK(cudaGetLastError());
  });
}

extern "C" int pe_allatonce_usolve(pe_ctx* c, const double* R, double* U, int nc, double* resid,
                                   void* stream) {
  return api_guard("pe_allatonce_usolve", [&] {
    require_arg(c && nc >= 0 && (nc == 0 || (R && U)), "need a context, nc >= 0 and buffers");
    PE_CUDA_CHECK(cudaSetDevice(c->device));
    allatonce_usolve(c, R, U, nc, resid, (cudaStream_t)stream);
  });
}

extern "C" int pe_wr_solver_residual(pe_ctx* c, double* out, void* stream) {
  return api_guard("pe_wr_solver_residual", [&] {
    require_arg(c && out, "need a context and an output buffer");
    if (!c->wr_ready || c->wr_last_nc < 1 || !c->Ux_cur.p)
      throw Error{PE_ERR_STATE, "no all-at-once solve to diagnose"};
    PE_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->d1 == 0) {
      PE_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(double) * c->E * c->wr_last_nc,
                                    (cudaStream_t)stream));
      return;
    }
    wr_solver_residual(c, out, (cudaStream_t)stream);
  });
}

extern "C" int pe_project_initial(int n, int d1, int d2, const int* M_ptr, const int* M_idx,
                                  const double* M_val, const int* P_colptr, const int* P_rowidx,
                                  const double* P_val, const double* M11, const double* M22,
                                  const double* u0, double* u_out, double* w_out, void* stream) {
  return api_guard("pe_project_initial", [&] {
    require_arg(n > 0 && d1 >= 0 && d2 >= 0 && M_ptr && P_colptr && u0,
                "need n > 0, d1, d2 >= 0 and buffers");
    require_arg((d1 == 0 || (M11 && u_out)) && (d2 == 0 || (M22 && w_out)), "NULL block");
    cudaStream_t st = (cudaStream_t)stream;
    const int d = d1 + d2;
    const int mnz = M_ptr[n], pnz = P_colptr[d];
    for (int i = 0; i < n; ++i) require_arg(M_ptr[i + 1] >= M_ptr[i], "bad CSR row pointers");
    for (int t = 0; t < mnz; ++t) require_arg(M_idx[t] >= 0 && M_idx[t] < n, "bad CSR column");
    for (int j = 0; j < d; ++j) require_arg(P_colptr[j + 1] >= P_colptr[j], "bad CSC pointers");
    for (int t = 0; t < pnz; ++t) require_arg(P_rowidx[t] >= 0 && P_rowidx[t] < n, "bad CSC row");
    Dev<int> mp(n + 1), mi(mnz), pp(d + 1), pi(pnz);
    Dev<double> mv(mnz), pv(pnz), x(n), v(n), b(d);
    auto up = [&](auto* dst, const auto* src, size_t cnt) {
      if (cnt)
        PE_CUDA_CHECK(cudaMemcpyAsync(dst, src, cnt * sizeof(*src), cudaMemcpyHostToDevice, st));
    };
    up(mp.p, M_ptr, n + 1);
    up(mi.p, M_idx, mnz);
    up(mv.p, M_val, mnz);
    up(pp.p, P_colptr, d + 1);
    up(pi.p, P_rowidx, pnz);
    up(pv.p, P_val, pnz);
    up(x.p, u0, n);
    k_csr_spmv<<<(n + 255) / 256, 256, 0, st>>>(n, mp.p, mi.p, mv.p, x.p, v.p);
    if (d) k_csc_tdot<<<(d + 7) / 8, 256, 0, st>>>(d, pp.p, pi.p, pv.p, v.p, b.p);
    g_launches += d ? 2 : 1;
    PE_CUDA_CHECK(cudaGetLastError());
    // M11 u = b1, M22 w = b2 by LU with partial pivoting (np.linalg.solve)
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS)
      throw Error{PE_ERR_SOLVER, "cusolverDnCreate failed"};
    struct HG {
      cusolverDnHandle_t h;
      ~HG() { cusolverDnDestroy(h); }
    } hg{h};
    cusolverDnSetStream(h, st);
    auto solve = [&](int m, const double* A_h, const double* rhs_dev, double* out_h) {
      if (!m) return;
      // row-major A = column-major A^T: solve A^T-stored system with trans = 'T'
      Dev<double> A((size_t)m * m), rb(m);
      Dev<int> piv(m), info(1);
      up(A.p, A_h, (size_t)m * m);
      PE_CUDA_CHECK(cudaMemcpyAsync(rb.p, rhs_dev, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
      int lw = 0;
      if (cusolverDnDgetrf_bufferSize(h, m, m, A.p, m, &lw) != CUSOLVER_STATUS_SUCCESS)
        throw Error{PE_ERR_SOLVER, "getrf buffer size failed"};
      Dev<double> work(lw > 0 ? lw : 1);
      if (cusolverDnDgetrf(h, m, m, A.p, m, work.p, piv.p, info.p) != CUSOLVER_STATUS_SUCCESS ||
          cusolverDnDgetrs(h, CUBLAS_OP_T, m, 1, A.p, m, piv.p, rb.p, m, info.p) !=
              CUSOLVER_STATUS_SUCCESS)
        throw Error{PE_ERR_SOLVER, "getrf/getrs failed"};
      int hinfo = 0;
      PE_CUDA_CHECK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaMemcpyAsync(out_h, rb.p, m * sizeof(double), cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      if (hinfo != 0) throw Error{PE_ERR_SOLVER, "singular coarse mass block"};
    };
    solve(d1, M11, b.p, u_out);
    solve(d2, M22, b.p + d1, w_out);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

extern "C" int pe_stability_max_step(pe_ctx* c, int member, double tol, int max_iter,
                                     double* bound, int* iterations, void* stream) {
  return api_guard("pe_stability_max_step", [&] {
    require_arg(c && bound && member >= 0 && member < c->E && max_iter >= 1 && tol > 0,
                "need a context, a member index, tol > 0, max_iter >= 1 and an output");
    PE_CUDA_CHECK(cudaSetDevice(c->device));
    const int n = c->d2;
    if (iterations) *iterations = 0;
    const double* A22 = c->A22.d() + (size_t)member * n * n;
    const double* M22 = c->M22.d() + (size_t)member * n * n;
    if (n == 0) {
      *bound = INFINITY;
      return;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // A22 == 0 (stepping.py:194): infinite bound
    {
      std::vector<double> h((size_t)n * n);
      PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), A22, sizeof(double) * h.size(),
                                    cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      double mx = 0.0;
      for (double x : h) mx = std::max(mx, std::fabs(x));
      if (mx == 0.0) {
        *bound = INFINITY;
        return;
      }
    }
    // P = M22^-1 A22 by Cholesky (cho_solve, stepping.py:199): potrs on the column-major
    // copies (M22 is symmetric, so its row-major storage is its column-major storage; A22 is
    // transposed into column-major on the host), then P back to row-major for the GEMV
    Dev<double> L((size_t)n * n), P((size_t)n * n), v(n), y(n), z(n), part(3 * 512);
    Dev<int> info(2);
    Dev<PowerState> ps(1);
    PE_CUDA_CHECK(cudaMemcpyAsync(L.p, M22, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
    {
      std::vector<double> h((size_t)n * n);
      PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), A22, sizeof(double) * h.size(),
                                    cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      std::vector<double> t((size_t)n * n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) t[(size_t)j * n + i] = h[(size_t)i * n + j];
      PE_CUDA_CHECK(cudaMemcpyAsync(P.p, t.data(), sizeof(double) * t.size(),
                                    cudaMemcpyHostToDevice, st));
      cusolverDnHandle_t h2 = nullptr;
      if (cusolverDnCreate(&h2) != CUSOLVER_STATUS_SUCCESS)
        throw Error{PE_ERR_SOLVER, "cusolverDnCreate failed"};
      struct HG {
        cusolverDnHandle_t h;
        ~HG() { cusolverDnDestroy(h); }
      } hg{h2};
      cusolverDnSetStream(h2, st);
      int lw = 0;
      cusolverDnDpotrf_bufferSize(h2, CUBLAS_FILL_MODE_LOWER, n, L.p, n, &lw);
      Dev<double> work(lw > 0 ? lw : 1);
      if (cusolverDnDpotrf(h2, CUBLAS_FILL_MODE_LOWER, n, L.p, n, work.p, lw, info.p) !=
              CUSOLVER_STATUS_SUCCESS ||
          cusolverDnDpotrs(h2, CUBLAS_FILL_MODE_LOWER, n, n, L.p, n, P.p, n, info.p + 1) !=
              CUSOLVER_STATUS_SUCCESS)
        throw Error{PE_ERR_SOLVER, "potrf/potrs failed"};
      int hi[2] = {0, 0};
      PE_CUDA_CHECK(cudaMemcpyAsync(hi, info.p, sizeof(hi), cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      if (hi[0] != 0) throw Error{PE_ERR_SOLVER, "M22 is not positive definite"};
      // X (column-major) = M22^-1 A22 = P: to row-major
      PE_CUDA_CHECK(cudaMemcpyAsync(t.data(), P.p, sizeof(double) * t.size(),
                                    cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[(size_t)i * n + j] = t[(size_t)j * n + i];
      PE_CUDA_CHECK(cudaMemcpyAsync(P.p, h.data(), sizeof(double) * h.size(),
                                    cudaMemcpyHostToDevice, st));
    }
    {
      std::vector<double> v0(n, 1.0 / std::sqrt((double)n));
      PE_CUDA_CHECK(cudaMemcpyAsync(v.p, v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
      PowerState p0{0.0, 0.0, 0, 0};
      PE_CUDA_CHECK(cudaMemcpyAsync(ps.p, &p0, sizeof(p0), cudaMemcpyHostToDevice, st));
    }
    const int nb = std::min(512, (n + 7) / 8);
    PowerState hp{};
    double* bufs[2] = {v.p, z.p};
    int it = 0;
    while (it < max_iter) {
      const int chunk = std::min(64, max_iter - it);
      for (int q = 0; q < chunk; ++q, ++it) {
        double* vin = bufs[it & 1];
        double* vout = bufs[(it + 1) & 1];
        k_pw_gemv<<<nb, 256, 0, st>>>(n, P.p, vin, y.p, part.p, ps.p);
        k_pw_rq<<<nb, 256, 0, st>>>(n, A22, M22, y.p, part.p, nb, vout, part.p + nb, ps.p);
        k_pw_finish<<<1, 1, 0, st>>>(nb, part.p + nb, tol, max_iter, ps.p);
        g_launches += 3;
      }
      PE_CUDA_CHECK(cudaGetLastError());
      PE_CUDA_CHECK(cudaMemcpyAsync(&hp, ps.p, sizeof(hp), cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      if (hp.done) break;
    }
    *bound = 2.0 / hp.lam;
    if (iterations) *iterations = hp.done == 1 ? hp.iters : -hp.iters;  // < 0: hit max_iter
  });
}
