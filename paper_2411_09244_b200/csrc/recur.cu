// Persistent cluster-resident recurrence kernel (the sequential-in-time chains).
//
//   mode WR  : W_s = E W_{s-1} + g_s, s = 0..J-1, W_{-1} = w0       (allatonce.py:226-229)
//   mode SEQ : X_{s+1} = T [X_s ; D_s] + c,  D_{s+1} = X_{s+1} - X_s, D_0 = 0
//              (stepping.py:122-147 x J, lags reset at the interval start :180)
//
// Interval columns are independent, so one thread-block cluster owns one (member,
// column group of 8 intervals) and walks all steps in a single launch.  Each CTA of the
// cluster keeps its 8-row-aligned slice of the stationary operator in shared memory
// for the whole launch; per step it computes its rows with FP64 DMMA (m8n8k4, K split
// across warps, partials reduced in a fixed order), publishes them through L2 and the
// cluster barrier orders the step.  No host round trip, no per-step launch.
// Column results do not depend on the column group they land in (batch invariance).

#include <cooperative_groups.h>

#include "pe.h"
#include "pe_internal.h"

namespace cg = cooperative_groups;

namespace pe {

constexpr int RC_THREADS = 256;
constexpr int RC_WARPS = RC_THREADS / 32;
constexpr int RC_CG = 8;  // interval columns per cluster (one n8 DMMA tile)

struct RecurArgs {
  int mode;        // 0 = WR, 1 = SEQ
  int M;           // output rows (d2 for WR, d for SEQ)
  int KT;          // operator columns (d2 for WR, 2d for SEQ)
  int nc;          // interval columns per member
  int S;           // steps
  int rpc;         // rows per CTA (multiple of 8)
  int cs;          // cluster size
  int ldo;         // operator row stride (= KT)
  const double* Op;
  long long op_b;  // per-member operator stride
  // WR: W (J+2 blocks of M x nc per member), block 1 = w0, block s+2 = g_s -> W_s
  double* W;
  long long w_b, L;
  // SEQ: X_in / X_out (E, nc, M), scratch Xs (2 x E x nc x 2M) for [X; D] exchange
  const double* Xin;
  double* Xout;
  double* Xs;
  const double* bias;
  long long bias_b;
};

__device__ __forceinline__ void dmma_rc(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int MT>  // m8 tiles per CTA (rpc = 8 * MT)
__global__ void __launch_bounds__(RC_THREADS) recur_kernel(const __grid_constant__ RecurArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / a.cs;
  const int ngroups = (a.nc + RC_CG - 1) / RC_CG;
  const int e = cid / ngroups, grp = cid - (cid / ngroups) * ngroups;
  const int r0 = rank * a.rpc;
  const int c0 = grp * RC_CG;
  const int KT = a.KT, M = a.M;
  const int SKO = KT + 4;  // padded row stride (doubles) of the operator slice / x columns
  extern __shared__ double sm[];
  double* opS = sm;                        // rpc x SKO
  double* xs = opS + (size_t)a.rpc * SKO;  // RC_CG x SKO  (x column-major by column)
  double* red = xs + (size_t)RC_CG * SKO;  // RC_WARPS x rpc x RC_CG
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  // operator slice -> smem (rows past M are zero)
  const double* Op = a.Op + (long long)e * a.op_b;
  for (int idx = tid; idx < a.rpc * KT; idx += RC_THREADS) {
    const int r = idx / KT, k = idx - (idx / KT) * KT;
    opS[r * SKO + k] = (r0 + r < M) ? Op[(long long)(r0 + r) * a.ldo + k] : 0.0;
  }
  // step-0 input: WR x = w0 (block 1 of W); SEQ [x; d] = [X_in; 0]
  double* Wm = nullptr;
  if (a.mode == 0) {
    Wm = a.W + (long long)e * a.w_b;
    const double* src = Wm + a.L;
    for (int idx = tid; idx < RC_CG * KT; idx += RC_THREADS) {
      const int c = idx / KT, k = idx - (idx / KT) * KT;
      xs[c * SKO + k] = (c0 + c < a.nc) ? __ldcg(src + (long long)(c0 + c) * M + k) : 0.0;
    }
  } else {
    const double* X0 = a.Xin + (long long)e * a.nc * M;
    for (int idx = tid; idx < RC_CG * KT; idx += RC_THREADS) {
      const int c = idx / KT, k = idx - (idx / KT) * KT;
      xs[c * SKO + k] = (c0 + c < a.nc && k < M) ? X0[(long long)(c0 + c) * M + k] : 0.0;
    }
  }
  const int Etot = gridDim.x / (a.cs * ngroups);
  __syncthreads();

  // split-K over warps, in multiples of 4
  const int kq = (KT + 3) / 4;
  const int kper = (kq + RC_WARPS - 1) / RC_WARPS;
  const int kb = warp * kper * 4, ke = min(KT, (warp + 1) * kper * 4);
  const double* bias = (a.mode == 1) ? a.bias + (long long)e * a.bias_b : nullptr;

  for (int s = 0; s < a.S; ++s) {
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    for (int k = kb; k < ke; k += 4) {
      const int kk = k + t4;
      const double b = (kk < KT) ? xs[g * SKO + kk] : 0.0;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const double av = (kk < KT) ? opS[(m * 8 + g) * SKO + kk] : 0.0;
        dmma_rc(acc[m][0], acc[m][1], av, b);
      }
    }
    // partial tile (row m*8+g, cols 2*t4, 2*t4+1) -> red[warp]
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      double* rw = red + ((size_t)warp * a.rpc + m * 8 + g) * RC_CG + 2 * t4;
      rw[0] = acc[m][0];
      rw[1] = acc[m][1];
    }
    __syncthreads();
    const bool last = (s == a.S - 1);
    for (int idx = tid; idx < a.rpc * RC_CG; idx += RC_THREADS) {
      const int r = idx / RC_CG, c = idx - (idx / RC_CG) * RC_CG;
      const int gr = r0 + r, gc = c0 + c;
      if (gr >= M || gc >= a.nc) continue;
      double v = 0.0;
      for (int w = 0; w < RC_WARPS; ++w) v += red[((size_t)w * a.rpc + r) * RC_CG + c];
      if (a.mode == 0) {
        double* dst = Wm + (long long)(s + 2) * a.L + (long long)gc * M + gr;
        v = __dadd_rn(v, *dst);  // + g_s  (w = E w + g, allatonce.py:228)
        *dst = v;
      } else {
        v = __dadd_rn(v, bias[gr]);
        const double xprev = xs[c * SKO + gr];
        if (last) {
          a.Xout[((long long)e * a.nc + gc) * M + gr] = v;
        } else {
          // exchange buffer: (2, E, nc, 2M), parity s&1; [X_{s+1}; D_{s+1}]
          double* xb = a.Xs + (((long long)(s & 1) * Etot + e) * a.nc + gc) * 2 * M;
          xb[gr] = v;
          xb[M + gr] = __dsub_rn(v, xprev);
        }
      }
    }
    cluster.sync();  // rows of step s published (release/acquire, cluster scope)
    if (!last) {
      if (a.mode == 0) {
        const double* src = Wm + (long long)(s + 2) * a.L;
        for (int idx = tid; idx < RC_CG * KT; idx += RC_THREADS) {
          const int c = idx / KT, k = idx - (idx / KT) * KT;
          xs[c * SKO + k] = (c0 + c < a.nc) ? __ldcg(src + (long long)(c0 + c) * M + k) : 0.0;
        }
      } else {
        const double* src = a.Xs + ((long long)(s & 1) * Etot + e) * a.nc * 2 * M;
        for (int idx = tid; idx < RC_CG * KT; idx += RC_THREADS) {
          const int c = idx / KT, k = idx - (idx / KT) * KT;
          xs[c * SKO + k] = (c0 + c < a.nc) ? __ldcg(src + (long long)(c0 + c) * 2 * M + k) : 0.0;
        }
      }
      __syncthreads();
    }
  }
}

// Plan: the largest cluster (<= 16 CTAs) whose 8-row-aligned operator slices cover M,
// provided a slice (plus x and the split-K scratch) fits in shared memory.
bool recur_plan(int M, int KT, int* rpc, int* cs, size_t* smem) {
  for (int c = 16; c >= 1; --c) {
    const int r = ((M + c - 1) / c + 7) / 8 * 8;
    const size_t bytes = sizeof(double) * ((size_t)r * (KT + 4) + (size_t)RC_CG * (KT + 4) +
                                           (size_t)RC_WARPS * r * RC_CG);
    if (r > 64 || bytes > 200 * 1024) return false;  // larger c only shrinks r
    *rpc = r;
    *cs = (M + r - 1) / r;
    *smem = bytes;
    return true;
  }
  return false;
}

template <int MT>
static void launch_recur(const RecurArgs& a, int E, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(recur_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       210 * 1024));
    PE_CUDA_CHECK(cudaFuncSetAttribute(recur_kernel<MT>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const int ngroups = (a.nc + RC_CG - 1) / RC_CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(E * ngroups * a.cs);
  cfg.blockDim = dim3(RC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = a.cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, recur_kernel<MT>, a));
  ++g_launches;
}

static void dispatch(const RecurArgs& a, int E, size_t smem, cudaStream_t st) {
  switch (a.rpc / 8) {
    case 1: launch_recur<1>(a, E, smem, st); break;
    case 2: launch_recur<2>(a, E, smem, st); break;
    case 3: launch_recur<3>(a, E, smem, st); break;
    case 4: launch_recur<4>(a, E, smem, st); break;
    case 5: launch_recur<5>(a, E, smem, st); break;
    case 6: launch_recur<6>(a, E, smem, st); break;
    case 7: launch_recur<7>(a, E, smem, st); break;
    case 8: launch_recur<8>(a, E, smem, st); break;
    default: throw Error{PE_ERR_ARG, "recurrence plan out of range"};
  }
}

bool recur_wr(int E, int d2, int nc, int J, const double* Emat, double* Wx, cudaStream_t st) {
  RecurArgs a{};
  size_t smem;
  if (!recur_plan(d2, d2, &a.rpc, &a.cs, &smem)) return false;
  a.mode = 0;
  a.M = d2;
  a.KT = d2;
  a.ldo = d2;
  a.nc = nc;
  a.S = J;
  a.Op = Emat;
  a.op_b = (long long)d2 * d2;
  a.L = (long long)d2 * nc;
  a.W = Wx;
  a.w_b = (long long)(J + 2) * a.L;
  dispatch(a, E, smem, st);
  return true;
}

bool recur_seq(int E, int d, int nc, int S, const double* T, const double* c, const double* Xin,
               double* Xout, double* scratch, cudaStream_t st) {
  RecurArgs a{};
  size_t smem;
  if (!recur_plan(d, 2 * d, &a.rpc, &a.cs, &smem)) return false;
  a.mode = 1;
  a.M = d;
  a.KT = 2 * d;
  a.ldo = 2 * d;
  a.nc = nc;
  a.S = S;
  a.Op = T;
  a.op_b = 2LL * d * d;
  a.Xin = Xin;
  a.Xout = Xout;
  a.Xs = scratch;  // 2 * E * nc * 2d doubles
  a.bias = c;
  a.bias_b = d;
  dispatch(a, E, smem, st);
  return true;
}

}  // namespace pe
