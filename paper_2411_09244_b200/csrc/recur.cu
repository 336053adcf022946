// Persistent cluster-resident recurrence kernel (the sequential-in-time chains).
//
//   mode WR  : W_s = E W_{s-1} + g_s, s = 0..J-1, W_{-1} = w0       (allatonce.py:226-229)
//   mode SEQ : X_{s+1} = T [X_s ; D_s] + c,  D_{s+1} = X_{s+1} - X_s, D_0 = 0
//              (stepping.py:122-147 x J, lags reset at the interval start :180)
//
// Interval columns are independent, so one thread-block cluster owns one (member,
// column group of 8 intervals) and walks all steps in a single launch.  Each CTA keeps its
// 8-row-aligned slice of the stationary operator in shared memory for the whole launch
// and computes its rows with FP64 DMMA (m8n8k4, K split across warps, partials reduced in
// a fixed order).  The new rows go point to point: 16-byte `st.async` remote stores into
// every peer's double-buffered x tile, each signalling the *receiver's* mbarrier
// (complete_tx).  A CTA waits only on its own mbarrier for the bytes of the step it
// consumes, so there is no cluster-wide barrier per step (B200 measurements:
// cluster.sync ~0.21 us; 13-way 8-byte DSMEM push + sync ~1.6 us per step).
// Column results do not depend on the column group they land in (batch invariance).

#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pe.h"
#include "pe_internal.h"
#include "mbar.cuh"

namespace cg = cooperative_groups;

namespace pe {

constexpr int RC_THREADS = 256;
constexpr int RC_WARPS = RC_THREADS / 32;
constexpr int RC_CG = 8;    // interval columns per cluster (one n8 DMMA tile)
constexpr int RC_CGP = 12;  // padded x row: 8 columns + 4 (conflict-free B fragments)

struct RecurArgs {
  int mode;        // 0 = WR, 1 = SEQ
  int M;           // output rows (d2 for WR, d for SEQ)
  int KT;          // operator columns (d2 for WR, 2d for SEQ)
  int KTP;         // KT padded to a multiple of 4 * RC_WARPS
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
  // SEQ: X_in / X_out (E, nc, M)
  const double* Xin;
  double* Xout;
  const double* bias;
  long long bias_b;
  unsigned long long* trace;  // optional phase timestamps (CTA 0, thread 0), debug only
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) \
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[slot] = gtimer();

__device__ __forceinline__ void dmma_rc(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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
  const int KT = a.KT, KTP = a.KTP, M = a.M;
  const int SKO = KTP + 4;  // operator row stride (doubles); +4 keeps A fragments conflict-free
  extern __shared__ __align__(16) double sm[];
  double* opS = sm;                                 // rpc x SKO
  double* xs2 = opS + (size_t)a.rpc * SKO;          // 2 x KTP x RC_CGP  (x[k][c], 2 buffers)
  double* red = xs2 + (size_t)2 * KTP * RC_CGP;     // RC_WARPS x rpc x RC_CG
  // step results staged for the bulk DSMEM copies: [2 parities][rpc][RC_CGP] (x, and d)
  double* ybuf2 = red + (size_t)RC_WARPS * a.rpc * RC_CG;
  double* dbuf2 = ybuf2 + (size_t)2 * a.rpc * RC_CGP;
  __shared__ __align__(8) unsigned long long mbar[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  TRACE(0)

  // operator slice -> smem (rows past M and columns past KT are zero), loads batched
  const double* Op = a.Op + (long long)e * a.op_b;
  for (int r = 0; r < a.rpc; r += 4) {
    double v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = tid + h * RC_THREADS;
        const bool ok = (r + u < a.rpc) && (r0 + r + u < M) && (k < KT);
        v[u][h] = ok ? __ldg(Op + (long long)(r0 + r + u) * a.ldo + k) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = tid + h * RC_THREADS;
        if (r + u < a.rpc && k < KTP) opS[(r + u) * SKO + k] = v[u][h];
      }
    for (int k = tid + 2 * RC_THREADS; k < KTP; k += RC_THREADS)  // KT > 512: plain loop
      for (int u = 0; u < 4 && r + u < a.rpc; ++u)
        opS[(r + u) * SKO + k] =
            (r0 + r + u < M && k < KT) ? __ldg(Op + (long long)(r0 + r + u) * a.ldo + k) : 0.0;
  }
  // step-0 input into buffer 0 (x[k][c]); buffer 1 zeroed (padding columns / k past KT)
  double* Wm = (a.mode == 0) ? a.W + (long long)e * a.w_b : nullptr;
  for (int idx = tid; idx < KTP * RC_CGP; idx += RC_THREADS) {
    const int k = idx / RC_CGP, c = idx - (idx / RC_CGP) * RC_CGP;
    double v = 0.0;
    if (c < RC_CG && c0 + c < a.nc && k < KT) {
      if (a.mode == 0)
        v = __ldcg(Wm + a.L + (long long)(c0 + c) * M + k);  // W_{-1} = w0 (block 1)
      else if (k < M)
        v = a.Xin[((long long)e * a.nc + c0 + c) * M + k];  // [X_0; D_0 = 0]
    }
    xs2[idx] = v;
    xs2[(size_t)KTP * RC_CGP + idx] = 0.0;
  }
  // one mbarrier per x buffer; bytes per phase = all M rows x 8 columns (x, and d for SEQ)
  const unsigned bytes = (unsigned)(M * RC_CGP * 8 * (a.mode == 1 ? 2 : 1));
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();  // barriers initialised and buffers zeroed before any peer pushes
  if (tid == 0) {  // arm: buffer 1 <- step-0 rows, buffer 0 <- step-1 rows
    mbar_expect_tx(smem_u32(&mbar[1]), bytes);
    if (a.S > 2) mbar_expect_tx(smem_u32(&mbar[0]), bytes);
  }
  TRACE(1)

  // split-K over warps (KTP is a multiple of 4 * RC_WARPS: no predicates in the loop)
  const int kper = KTP / RC_WARPS;
  const int kb = warp * kper;
  const double* bias = (a.mode == 1) ? a.bias + (long long)e * a.bias_b : nullptr;
  constexpr int OUT_PER_T = (8 * MT * RC_CG + RC_THREADS - 1) / RC_THREADS;
  const unsigned xs_base = smem_u32(xs2);
  const unsigned bar_base = smem_u32(&mbar[0]);

  for (int s = 0; s < a.S; ++s) {
    const int cur = s & 1;
    const double* xs = xs2 + (size_t)cur * KTP * RC_CGP;
    double* ybuf = ybuf2 + (size_t)cur * a.rpc * RC_CGP;
    double* dbuf = dbuf2 + (size_t)cur * a.rpc * RC_CGP;
    // the bulk copies issued two steps ago read this parity's staging buffer: done?
    if (tid < a.cs) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (s > 0) {
      mbar_wait(bar_base + 8 * cur, ((s - 1) >> 1) & 1);
      // re-arm this buffer for the rows of step s+1 (consumed at step s+2)
      if (tid == 0 && s + 2 < a.S) mbar_expect_tx(bar_base + 8 * cur, bytes);
    }
    TRACE(2 + 4 * s)
    double gpre[OUT_PER_T];
    if (a.mode == 0) {  // g_s for this thread's outputs, fetched under the DMMA work
#pragma unroll
      for (int u = 0; u < OUT_PER_T; ++u) {
        const int idx = tid + u * RC_THREADS;
        const int r = idx >> 3, c = idx & 7;
        gpre[u] = (idx < a.rpc * RC_CG && r0 + r < M && c0 + c < a.nc)
                      ? __ldcg(Wm + (long long)(s + 2) * a.L + (long long)(c0 + c) * M + r0 + r)
                      : 0.0;
      }
    }
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    const double* xb = xs + (size_t)(kb + t4) * RC_CGP + g;
    const double* ob = opS + (size_t)g * SKO + kb + t4;
#pragma unroll 4
    for (int k = 0; k < kper; k += 4) {
      const double b = xb[(size_t)k * RC_CGP];
#pragma unroll
      for (int m = 0; m < MT; ++m) dmma_rc(acc[m][0], acc[m][1], ob[(size_t)m * 8 * SKO + k], b);
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      double* rw = red + ((size_t)warp * a.rpc + m * 8 + g) * RC_CG + 2 * t4;
      rw[0] = acc[m][0];
      rw[1] = acc[m][1];
    }
    __syncthreads();
    TRACE(3 + 4 * s)
    const bool last = (s == a.S - 1);
    // fixed-order reduction over warps + epilogue, one (row, column) per thread
#pragma unroll
    for (int u = 0; u < OUT_PER_T; ++u) {
      const int idx = tid + u * RC_THREADS;
      if (idx >= a.rpc * RC_CG) continue;
      const int r = idx >> 3, c = idx & 7;
      const int gr = r0 + r, gc = c0 + c;
      double v = 0.0;
      for (int w = 0; w < RC_WARPS; ++w) v += red[((size_t)w * a.rpc + r) * RC_CG + c];
      double dv = 0.0;
      if (gr < M) {
        if (a.mode == 0) {
          v = __dadd_rn(v, gpre[u]);  // + g_s  (w = E w + g, allatonce.py:228)
          if (gc < a.nc) Wm[(long long)(s + 2) * a.L + (long long)gc * M + gr] = v;
        } else {
          v = __dadd_rn(v, bias[gr]);
          dv = __dsub_rn(v, xs[(size_t)gr * RC_CGP + c]);  // D_{s+1} = X_{s+1} - X_s
          if (last && gc < a.nc) a.Xout[((long long)e * a.nc + gc) * M + gr] = v;
        }
        if (gc >= a.nc) v = dv = 0.0;  // padding columns stay zero
      }
      ybuf[r * RC_CGP + c] = v;
      dbuf[r * RC_CGP + c] = dv;
    }
    if (!last) {
      // push: one bulk DSMEM copy per peer (and per d block for SEQ) of this CTA's row block
      // into the peer's next x buffer, completing on the peer's mbarrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid < a.cs) {
        const int q = tid;
        const int nrow = min(a.rpc, M - r0);
        const unsigned nbuf = xs_base + (unsigned)(((s + 1) & 1) * KTP * RC_CGP * 8);
        const unsigned rbar = map_rank(bar_base + 8 * ((s + 1) & 1), q);
        const unsigned bytes_blk = (unsigned)(nrow * RC_CGP * 8);
        const unsigned dst = map_rank(nbuf + (unsigned)(r0 * RC_CGP * 8), q);
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst), "r"(smem_u32(ybuf)), "r"(bytes_blk), "r"(rbar) : "memory");
        if (a.mode == 1) {
          const unsigned dd = map_rank(nbuf + (unsigned)((M + r0) * RC_CGP * 8), q);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(dd), "r"(smem_u32(dbuf)), "r"(bytes_blk), "r"(rbar) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    TRACE(4 + 4 * s)
    TRACE(5 + 4 * s)
  }
  if (tid < a.cs) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  cluster.sync();  // no CTA leaves while copies to or from it may be in flight
}

static size_t recur_smem(int r, int KTP) {
  return sizeof(double) * ((size_t)r * (KTP + 4) + 2 * (size_t)KTP * RC_CGP +
                           (size_t)RC_WARPS * r * RC_CG + 4 * (size_t)r * RC_CGP);
}

static int pad_k(int KT) { return (KT + 4 * RC_WARPS - 1) / (4 * RC_WARPS) * (4 * RC_WARPS); }

template <int MT>
static void set_attrs() {
  static bool done = false;
  if (!done) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(recur_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       210 * 1024));
    PE_CUDA_CHECK(cudaFuncSetAttribute(recur_kernel<MT>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    done = true;
  }
}

template <int MT>
static int max_active_clusters(int cs, size_t smem) {
  set_attrs<MT>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(RC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, recur_kernel<MT>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static int active_clusters(int rpc, int cs, size_t smem) {
  switch (rpc / 8) {
    case 1: return max_active_clusters<1>(cs, smem);
    case 2: return max_active_clusters<2>(cs, smem);
    case 3: return max_active_clusters<3>(cs, smem);
    case 4: return max_active_clusters<4>(cs, smem);
    case 5: return max_active_clusters<5>(cs, smem);
    case 6: return max_active_clusters<6>(cs, smem);
    case 7: return max_active_clusters<7>(cs, smem);
    case 8: return max_active_clusters<8>(cs, smem);
  }
  return 0;
}

// Plan: 8-row-aligned slices over <= 16 CTAs whose operator slice, x double buffer and
// split-K scratch fit in shared memory.  Clusters must fit inside a GPC, so the number of
// co-resident clusters depends on (cluster size, smem); pick the plan with the fewest
// waves of `nclusters`, then the thinnest slice (least DMMA work per step).
bool recur_plan(int M, int KT, int* rpc, int* cs, size_t* smem, int nclusters) {
  const int KTP = pad_k(KT);
  int best_w = 1 << 30, best_r = 0;
  for (int r = ((M + 15) / 16 + 7) / 8 * 8; r <= 64; r += 8) {
    const size_t bytes = recur_smem(r, KTP);
    if (bytes > 200 * 1024) break;
    const int c = (M + r - 1) / r;
    int act = 1;
    if (nclusters > 0) {
      act = active_clusters(r, c, bytes);
      if (act <= 0) continue;
    }
    const int waves = nclusters > 0 ? (nclusters + act - 1) / act : 1;
    if (waves < best_w) {
      best_w = waves;
      best_r = r;
    }
    if (nclusters <= 0 || waves == 1) break;
  }
  if (best_r == 0) return false;
  *rpc = best_r;
  *cs = (M + best_r - 1) / best_r;
  *smem = recur_smem(best_r, KTP);
  return true;
}

template <int MT>
static void launch_recur(const RecurArgs& a, int E, size_t smem, cudaStream_t st) {
  set_attrs<MT>();
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

static void run_traced(RecurArgs& a, int E, size_t smem, cudaStream_t st, const char* tag) {
  static const bool trace = getenv("PE_RECUR_TRACE") != nullptr;
  unsigned long long* tb = nullptr;
  const int n = 2 + 4 * a.S + 8;
  if (trace) {
    PE_CUDA_CHECK(cudaMalloc(&tb, sizeof(unsigned long long) * n));
    PE_CUDA_CHECK(cudaMemset(tb, 0, sizeof(unsigned long long) * n));
  }
  a.trace = tb;
  dispatch(a, E, smem, st);
  if (trace) {
    std::vector<unsigned long long> h(n);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    PE_CUDA_CHECK(cudaMemcpy(h.data(), tb, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
    double wait = 0, mma = 0, epi = 0;
    for (int s = 0; s < a.S; ++s) {
      if (s > 0) wait += (h[2 + 4 * s] - h[4 + 4 * (s - 1)]) * 1e-3;
      mma += (h[3 + 4 * s] - h[2 + 4 * s]) * 1e-3;
      epi += (h[4 + 4 * s] - h[3 + 4 * s]) * 1e-3;
    }
    fprintf(stderr,
            "recur %s trace (cs=%d rpc=%d): setup %.2f us, per step: wait %.3f mma %.3f "
            "epi+push %.3f us, total %.2f us\n",
            tag, a.cs, a.rpc, (h[1] - h[0]) * 1e-3, wait / a.S, mma / a.S, epi / a.S,
            (h[5 + 4 * (a.S - 1)] - h[0]) * 1e-3);
    cudaFree(tb);
  }
}

bool recur_wr(int E, int d2, int nc, int J, const double* Emat, double* Wx, cudaStream_t st) {
  RecurArgs a{};
  size_t smem;
  if (!recur_plan(d2, d2, &a.rpc, &a.cs, &smem, E * ((nc + RC_CG - 1) / RC_CG))) return false;
  a.mode = 0;
  a.M = d2;
  a.KT = d2;
  a.KTP = pad_k(d2);
  a.ldo = d2;
  a.nc = nc;
  a.S = J;
  a.Op = Emat;
  a.op_b = (long long)d2 * d2;
  a.L = (long long)d2 * nc;
  a.W = Wx;
  a.w_b = (long long)(J + 2) * a.L;
  run_traced(a, E, smem, st, "wr");
  return true;
}

bool recur_seq(int E, int d, int nc, int S, const double* T, const double* c, const double* Xin,
               double* Xout, double* /*scratch*/, cudaStream_t st) {
  RecurArgs a{};
  size_t smem;
  if (!recur_plan(d, 2 * d, &a.rpc, &a.cs, &smem, E * ((nc + RC_CG - 1) / RC_CG))) return false;
  a.mode = 1;
  a.M = d;
  a.KT = 2 * d;
  a.KTP = pad_k(2 * d);
  a.ldo = 2 * d;
  a.nc = nc;
  a.S = S;
  a.Op = T;
  a.op_b = 2LL * d * d;
  a.Xin = Xin;
  a.Xout = Xout;
  a.bias = c;
  a.bias_b = d;
  run_traced(a, E, smem, st, "seq");
  return true;
}

}  // namespace pe
