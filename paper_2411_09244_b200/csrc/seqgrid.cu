// Persistent all-SM kernel for the sequential fine propagator when the step operator is too
// large for one thread-block cluster's shared memory (cfg2: T is 600 x 1200 = 5.8 MB).
//
//   X_{s+1} = T [X_s ; D_s] + c,   D_{s+1} = X_{s+1} - X_s,  D_0 = 0
//   (stepping.py:122-147 x J, lags reset at the interval start :180)
//
// Layout.  The state of all interval columns lives in L2 as Z[parity][column][2d] in the
// permuted order [X (d) ; Dw (d2) ; Du (d1)]: the u rows of T do not touch Du (the split
// step's u-solve uses w - w_prev only, stepping.py:131), so u-row tiles contract over the
// first d + d2 entries and w-row tiles over all 2d.  One CTA per SM owns a (row tile x column
// group) block of the output: its slice of T stays in shared memory for all J steps, the
// column group's Z is streamed from L2 every step.
//
// Step protocol (no grid-wide barrier).  A CTA publishes its rows of step s by a release
// increment of its column group's counter; step s+1 of that group starts once the counter
// reaches (s+1) x (row tiles).  Z is double buffered by step parity; a CTA overwrites parity
// p only after every CTA of its group has finished the step that read p (the counter wait
// orders that).  Column groups never interact.
//
// Inner loop.  K is split over the 8 warps; each warp streams its own K slice of Z through a
// private 2-stage cp.async ring (no CTA barrier in the main loop) and accumulates all
// (rows/8) x (cols/8) DMMA m8n8k4 tiles of the block.  Warp partials are summed in a fixed
// order: the result is deterministic and independent of the launch plan's column grouping.

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pe.h"
#include "pe_internal.h"

namespace pe {

constexpr int SG_THREADS = 256;  // two warps per SMSP (one warp cannot hide LDS + pipeline overhead)
constexpr int SG_WARPS = SG_THREADS / 32;
constexpr int SG_KCH = 16;     // k per pipeline chunk
constexpr int SG_STAGES = 2;   // per-warp ring depth
constexpr int SG_MAXR = 148;   // row tiles per column group (<= SMs)
constexpr int SG_MT = 3;       // max m8 tiles (rows / 8) per CTA

struct SeqGridArgs {
  int d, d1, d2, nc, S;
  int ct;                      // columns per group (multiple of 8)
  int R;                       // row tiles per column group
  int tsmax;                   // largest T slice over tiles, doubles (rows x (KP + 4))
  unsigned long long* trace;   // optional per-step phase timestamps (CTA 0), debug only
  short r0[SG_MAXR], rows[SG_MAXR], kp[SG_MAXR], kt[SG_MAXR];
  const double* T;             // d x 2d row-major, columns [X ; Du ; Dw]
  const double* bias;          // d
  double* Z;                   // 2 x nc x 2d, permuted [X ; Dw ; Du]
  double* Xout;                // nc x d
  unsigned* cnt;               // one monotonic counter per column group
};

__device__ __forceinline__ void sg_cp16(unsigned dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void sg_dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned long long sg_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SG_TRACE(slot) \
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[slot] = sg_timer();

__device__ __forceinline__ unsigned sg_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// column k of the permuted contraction -> column of T's [X ; Du ; Dw] layout
__device__ __forceinline__ int sg_tcol(int k, int d, int d1, int d2) {
  if (k < d) return k;
  if (k < d + d2) return d + d1 + (k - d);  // Dw
  return d + (k - d - d2);                  // Du
}

template <int NT>
__global__ void __launch_bounds__(SG_THREADS, 1) seqgrid_kernel(const __grid_constant__ SeqGridArgs a) {
  const int cg = blockIdx.x / a.R, rt = blockIdx.x - (blockIdx.x / a.R) * a.R;
  const int r0 = a.r0[rt], RT = a.rows[rt], KP = a.kp[rt], KT = a.kt[rt];
  const int mt = RT >> 3;
  const int c0 = cg * a.ct;
  const int ncol = min(a.ct, a.nc - c0);
  const int d = a.d, d1 = a.d1, d2 = a.d2, D2 = 2 * d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr int CT = NT * 8;
  constexpr int ZS = SG_KCH + 4;                   // ring row stride (col-major chunk)
  const int SKO = KP + 4;                          // T slice row stride (conflict-free A)
  extern __shared__ __align__(16) double sm[];
  double* Ts = sm;                                 // RT x SKO
  double* ring = sm + a.tsmax;                     // warps x stages x CT x ZS
  constexpr int PS = CT + 8;                       // partial row stride: conflict-free double2
  constexpr int WREG = (SG_STAGES * CT * ZS > SG_MT * 8 * PS) ? SG_STAGES * CT * ZS : SG_MT * 8 * PS;
  double* myring = ring + (size_t)warp * WREG;     // ring, then this warp's partial tile

  // T slice -> smem in contraction order; rows past d and k past KT are zero
  for (int idx = tid; idx < RT * KP; idx += SG_THREADS) {
    const int r = idx / KP, k = idx - (idx / KP) * KP;
    const int gr = r0 + r;
    double v = 0.0;
    if (gr < d && k < KT) v = __ldg(a.T + (size_t)gr * D2 + sg_tcol(k, d, d1, d2));
    Ts[(size_t)r * SKO + k] = v;
  }
  __syncthreads();

  // this warp's K slice, in whole chunks
  const int nch = KP / SG_KCH;
  const int cb = (warp * nch) / SG_WARPS, ce = ((warp + 1) * nch) / SG_WARPS;

  SG_TRACE(0)
  for (int s = 0; s < a.S; ++s) {
    const int p = s & 1;
    SG_TRACE(1 + 4 * s)
    if (s > 0) {
      if (tid == 0) {
        const unsigned target = (unsigned)s * (unsigned)a.R;
        while (sg_ld_acquire(a.cnt + cg) < target) {
        }
      }
      __syncthreads();
    }
    SG_TRACE(2 + 4 * s)
    const double* Zp = a.Z + ((size_t)p * a.nc + c0) * D2;
    auto load_chunk = [&](int ch, int slot) {
      double* dst = myring + (size_t)slot * CT * ZS;
      const int k0 = ch * SG_KCH;
      // CT columns x 16 k = CT x 8 sixteen-byte pieces; 32 lanes
#pragma unroll
      for (int i = 0; i < (CT * 8 + 31) / 32; ++i) {
        const int q = lane + i * 32;
        if (q < CT * 8) {
          const int col = q >> 3, kk = (q & 7) * 2;
          const int k = k0 + kk;
          const bool ok = col < ncol && k < KT;
          const double* src = ok ? Zp + (size_t)col * D2 + k : Zp;
          sg_cp16((unsigned)__cvta_generic_to_shared(dst + col * ZS + kk), src, ok ? 16 : 0);
        }
      }
    };
#pragma unroll
    for (int i = 0; i < SG_STAGES - 1; ++i) {  // prologue: STAGES-1 chunks in flight
      if (cb + i < ce) load_chunk(cb + i, i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    // epilogue operands of this thread's outputs, fetched under the main loop: X_s of the
    // output rows (for D_{s+1}) and the bias
    constexpr int OPT = (SG_MT * 8 * CT + SG_THREADS - 1) / SG_THREADS;
    double xo[OPT], bo[OPT];
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int idx = tid + u * SG_THREADS;
      const int r = idx / CT, c = idx - (idx / CT) * CT;
      const bool ok = idx < RT * CT && r0 + r < d && c < ncol;
      xo[u] = ok ? __ldcg(Zp + (size_t)c * D2 + r0 + r) : 0.0;
      bo[u] = ok ? __ldg(a.bias + r0 + r) : 0.0;
    }
    double acc[SG_MT][NT][2];
#pragma unroll
    for (int m = 0; m < SG_MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    // main loop specialised on the CTA's row-tile count (uniform per CTA): a runtime guard
    // around each DMMA would predicate the warp-synchronous MMAs (WARPSYNC + NOP per group)
    auto mainloop = [&](auto MTC) {
      constexpr int MTK = decltype(MTC)::value;
      for (int ch = cb; ch < ce; ++ch) {
        const int i = ch - cb, slot = i % SG_STAGES;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(SG_STAGES - 2) : "memory");  // chunk ch landed
        __syncwarp();  // ... for every lane; and slot (i-1) % STAGES is no longer read
        if (ch + SG_STAGES - 1 < ce) load_chunk(ch + SG_STAGES - 1, (i + SG_STAGES - 1) % SG_STAGES);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const double* zs = myring + (size_t)slot * CT * ZS + g * ZS + t4;
        const double* ts = Ts + (size_t)g * SKO + ch * SG_KCH + t4;
#pragma unroll
        for (int kk = 0; kk < SG_KCH; kk += 4) {
          double bf[NT], af[MTK];
#pragma unroll
          for (int n = 0; n < NT; ++n) bf[n] = zs[n * 8 * ZS + kk];
#pragma unroll
          for (int m = 0; m < MTK; ++m) af[m] = ts[(size_t)m * 8 * SKO + kk];
#pragma unroll
          for (int m = 0; m < MTK; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) sg_dmma(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
        }
      }
    };
    if (mt == 3)
      mainloop(std::integral_constant<int, 3>{});
    else if (mt == 2)
      mainloop(std::integral_constant<int, 2>{});
    else
      mainloop(std::integral_constant<int, 1>{});
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    SG_TRACE(3 + 4 * s)
    // warp partial -> own region ([r][c], stride PS; one 16-byte store per fragment pair)
#pragma unroll
    for (int m = 0; m < SG_MT; ++m)
      if (m < mt)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          *reinterpret_cast<double2*>(myring + (size_t)(m * 8 + g) * PS + n * 8 + 2 * t4) =
              make_double2(acc[m][n][0], acc[m][n][1]);
    __syncthreads();
    // fixed-order reduction over warps + epilogue, one (row, column) per thread
    double* Zn = a.Z + ((size_t)(p ^ 1) * a.nc + c0) * D2;
    const bool last = (s == a.S - 1);
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int idx = tid + u * SG_THREADS;
      const int r = idx / CT, c = idx - (idx / CT) * CT;
      const int gr = r0 + r;
      if (idx >= RT * CT || gr >= d || c >= ncol) continue;
      double v = 0.0;
      for (int w = 0; w < SG_WARPS; ++w)
        v += ring[(size_t)w * WREG + (size_t)r * PS + c];
      v = __dadd_rn(v, bo[u]);
      const double dv = __dsub_rn(v, xo[u]);  // D_{s+1} = X_{s+1} - X_s
      double* zc = Zn + (size_t)c * D2;
      __stcg(zc + gr, v);
      __stcg(zc + (gr < d1 ? d + d2 + gr : d + (gr - d1)), dv);
      if (last) a.Xout[(size_t)(c0 + c) * d + gr] = v;
    }
    // publish: CTA barrier, then one gpu-scope release increment (the barrier orders every
    // thread's stores before it; same pattern as a cooperative-groups grid barrier)
    __syncthreads();
    if (tid == 0)  // release at gpu scope: orders the CTA's stores (via the barrier) first
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.cnt + cg) : "memory");
    SG_TRACE(4 + 4 * s)
  }
}

__global__ void seqgrid_init_kernel(int d, int nc, const double* __restrict__ Xin, double* Z) {
  const long long D2 = 2LL * d, total = (long long)nc * D2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long n = t / D2;
    const int k = (int)(t - n * D2);
    Z[t] = (k < d) ? Xin[n * d + k] : 0.0;  // [X_0 ; D_0 = 0]
  }
}

struct SeqGridPlan {
  bool ok = false;
  int ct = 0, ncg = 0, R = 0;
  size_t tsmax = 0, smem = 0;
  long long cost = 0;
  short r0[SG_MAXR], rows[SG_MAXR], kp[SG_MAXR], kt[SG_MAXR];
};

static size_t sg_smem(size_t tsmax, int ct) {
  const size_t ring = (size_t)SG_STAGES * ct * (SG_KCH + 4), part = (size_t)SG_MT * 8 * (ct + 8);
  return sizeof(double) * (tsmax + (size_t)SG_WARPS * std::max(ring, part));
}

static int sg_pad(int k) { return (k + SG_KCH - 1) / SG_KCH * SG_KCH; }

// Pack 8-row strips into <= R contiguous row tiles whose DMMA count per step stays <= cap.
static bool sg_pack(int d, int d1, int d2, int ct, int R, long long cap, size_t smem_cap,
                    SeqGridPlan& pl) {
  const int nstrip = (d + 7) / 8;
  const int Ku = d + d2, Kw = 2 * d;
  int t = 0, s = 0;
  size_t tsmax = 0;
  while (s < nstrip) {
    if (t >= R) return false;
    int rows = 0, K = 0;
    int e = s;
    while (e < nstrip) {
      const int kk = (8 * (e + 1) <= d1) ? Ku : Kw;
      const int K2 = std::max(K, kk);
      const int rows2 = rows + 8;
      const long long cost = (long long)(rows2 / 8) * (ct / 8) * (sg_pad(K2) / 4);
      const size_t ts2 = std::max(tsmax, (size_t)rows2 * (sg_pad(K2) + 4));
      if (rows2 / 8 > SG_MT || cost > cap || sg_smem(ts2, ct) > smem_cap) break;
      rows = rows2;
      K = K2;
      ++e;
    }
    if (e == s) return false;
    pl.r0[t] = (short)(8 * s);
    pl.rows[t] = (short)rows;
    pl.kt[t] = (short)K;
    pl.kp[t] = (short)sg_pad(K);
    tsmax = std::max(tsmax, (size_t)rows * (sg_pad(K) + 4));
    ++t;
    s = e;
  }
  pl.R = t;
  pl.tsmax = tsmax;
  return true;
}

static bool seqgrid_plan(int d1, int d2, int nc, SeqGridPlan& best) {
  const int d = d1 + d2;
  if (d <= 0 || nc <= 0 || d > 8000) return false;
  const size_t smem_cap = 220 * 1024;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sms = std::min(v, SG_MAXR);
  }
  best.ok = false;
  for (int ct = 8; ct <= 32; ct += 8) {
    const int ncg = (nc + ct - 1) / ct;
    const int R = sms / ncg;
    if (R < 1) continue;
    // smallest per-CTA DMMA cap that packs into R row tiles
    long long lo = 1, hi = (long long)SG_MT * (ct / 8) * (sg_pad(2 * d) / 4);
    SeqGridPlan pl;
    if (!sg_pack(d, d1, d2, ct, R, hi, smem_cap, pl)) continue;
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      SeqGridPlan t;
      if (sg_pack(d, d1, d2, ct, R, mid, smem_cap, t))
        hi = mid;
      else
        lo = mid + 1;
    }
    sg_pack(d, d1, d2, ct, R, hi, smem_cap, pl);
    pl.ct = ct;
    pl.ncg = ncg;
    pl.cost = hi;
    pl.smem = sg_smem(pl.tsmax, ct);
    pl.ok = true;
    if (!best.ok || pl.cost < best.cost ||
        (pl.cost == best.cost && pl.ncg * pl.R < best.ncg * best.R))
      best = pl;
  }
  return best.ok;
}

bool seqgrid_fits(int E, int d1, int d2, int nc) {
  if (E != 1) return false;
  SeqGridPlan pl;
  return seqgrid_plan(d1, d2, nc, pl);
}

template <int NT>
static void launch_sg(const SeqGridArgs& a, int grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(seqgrid_kernel<NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, seqgrid_kernel<NT>, a));
  ++g_launches;
}

bool seqgrid_seq(int d1, int d2, int nc, int S, const double* T, const double* c,
                 const double* Xin, double* Xout, double* Z, unsigned* cnt, cudaStream_t st) {
  SeqGridPlan pl;
  if (!seqgrid_plan(d1, d2, nc, pl)) return false;
  const int d = d1 + d2;
  const long long total = 2LL * d * nc;
  seqgrid_init_kernel<<<(int)std::min<long long>(148 * 4, (total + 255) / 256), 256, 0, st>>>(
      d, nc, Xin, Z);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  PE_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * pl.ncg, st));
  SeqGridArgs a{};
  a.d = d;
  a.d1 = d1;
  a.d2 = d2;
  a.nc = nc;
  a.S = S;
  a.ct = pl.ct;
  a.R = pl.R;
  a.tsmax = (int)pl.tsmax;
  for (int i = 0; i < pl.R; ++i) {
    a.r0[i] = pl.r0[i];
    a.rows[i] = pl.rows[i];
    a.kp[i] = pl.kp[i];
    a.kt[i] = pl.kt[i];
  }
  a.T = T;
  a.bias = c;
  a.Z = Z;
  a.Xout = Xout;
  a.cnt = cnt;
  static const bool trace = getenv("PE_SEQGRID_TRACE") != nullptr;
  if (trace)
    fprintf(stderr, "seqgrid plan: ct=%d ncg=%d R=%d ctas=%d smem=%zu cost=%lld\n", pl.ct,
            pl.ncg, pl.R, pl.ncg * pl.R, pl.smem, pl.cost);
  const int grid = pl.ncg * pl.R;
  const int ntr = 2 + 4 * S;
  if (trace) {
    PE_CUDA_CHECK(cudaMalloc(&a.trace, sizeof(unsigned long long) * ntr));
    PE_CUDA_CHECK(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * ntr, st));
  }
  switch (pl.ct / 8) {
    case 1: launch_sg<1>(a, grid, pl.smem, st); break;
    case 2: launch_sg<2>(a, grid, pl.smem, st); break;
    case 3: launch_sg<3>(a, grid, pl.smem, st); break;
    default: launch_sg<4>(a, grid, pl.smem, st); break;
  }
  if (trace) {
    std::vector<unsigned long long> h(ntr);
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    PE_CUDA_CHECK(cudaMemcpy(h.data(), a.trace, sizeof(unsigned long long) * ntr,
                             cudaMemcpyDeviceToHost));
    double wait = 0, mma = 0, epi = 0;
    for (int s = 0; s < S; ++s) {
      wait += (h[2 + 4 * s] - h[1 + 4 * s]) * 1e-3;
      mma += (h[3 + 4 * s] - h[2 + 4 * s]) * 1e-3;
      epi += (h[4 + 4 * s] - h[3 + 4 * s]) * 1e-3;
    }
    fprintf(stderr, "seqgrid trace: setup %.2f us, per step wait %.3f mainloop %.3f epi %.3f us, "
            "total %.1f us\n", (h[1] - h[0]) * 1e-3, wait / S, mma / S, epi / S,
            (h[4 + 4 * (S - 1)] - h[0]) * 1e-3);
    cudaFree(a.trace);
  }
  return true;
}

}  // namespace pe
