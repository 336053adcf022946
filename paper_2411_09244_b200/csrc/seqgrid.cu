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
// range) block of the output: its slice of T stays in shared memory for all J steps, the
// columns' Z is streamed from L2 every step.
//
// Step protocol (no grid-wide barrier).  The columns of a CTA's range are split into H chain
// groups (8..32 interval columns each) that the CTA steps round-robin: sub-step i = (s, h) is
// step s of group h.  A CTA publishes its rows of a sub-step by a release increment of the
// group's counter; step s+1 of the group starts once the counter reaches (s+1) x (row tiles).
// Z is double buffered by step parity; a CTA overwrites parity p only after every CTA of the
// group has finished the step that read p (the counter wait orders that).  Chain groups never
// interact.
//
// The exchange runs beside the arithmetic.  Two extra warps own the two ends of the protocol:
// the admit warp polls the counter of the next sub-step and posts "ready" in shared memory;
// the publish warp waits for the compute warps' stores of a finished sub-step (mbarrier) and
// does the gpu-scope release increment -- so the fence, the L2 round trips of the poll and the
// other CTAs' skew are covered by the compute of the CTA's other chain groups.  The compute warps
// never wait on global memory state; when the next sub-step is already "ready" at the tail of
// a main loop they stream its first Z chunks into the ring slots that fall free.
//
// Inner loop.  K is split over the 8 compute warps; each warp streams its own K slice of Z
// through a private cp.async ring (no CTA barrier in the main loop) and accumulates all
// (rows/8) x (cols/8) DMMA m8n8k4 tiles of the block.  Warp partials are summed in a fixed
// order: the result is deterministic and independent of the launch plan's column grouping.

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pe.h"
#include "pe_internal.h"
#include "mbar.cuh"

namespace pe {

// Build-time knobs of the measured variants (cfg2-seq, us per chain step, B200):
//   8 warps x 16-k chunks x 4 stages 5.32 (kept) | 8 x 8 6.68 | 12 x 8 5.87 | 8 x 24 x 3 5.47 |
//   8 x 32 x 2 5.33 | 8 x 16 x 3 5.33.  The critical warp runs ~49 cycles per DMMA whatever
//   the chunk size: two warps per SMSP share the DMMA pipe (16 cycles each) and the
//   shared-memory pipe, which moves T slice + Z reads + Z writes = 292 KB per sub-step
//   (84 % of the 128 B/clk x 1.42 us the DMMAs need).
#ifndef SG_CWARPS_N
#define SG_CWARPS_N 8
#endif
#ifndef SG_KCH_N
#define SG_KCH_N 16
#endif
constexpr int SG_CWARPS = SG_CWARPS_N;  // compute warps (one per SMSP cannot hide LDS + pipeline overhead)
constexpr int SG_CTHREADS = SG_CWARPS * 32;
constexpr int SG_THREADS = SG_CTHREADS + 64;  // + the admit warp and the publish warp
constexpr int SG_WARPS = SG_CWARPS;
constexpr int SG_KCH = SG_KCH_N;  // k per pipeline chunk
constexpr int SG_MAXR = 148;   // row tiles per column range (<= SMs)
constexpr int SG_MT = 3;       // max m8 tiles (rows / 8) per CTA
constexpr int SG_MAXH = 4;     // chain groups per CTA
// per-warp ring depth: 8-column chain groups leave room for four stages
#ifndef SG_STG1
#define SG_STG1 4
#endif
__host__ __device__ constexpr int sg_stages(int nt) { return nt == 1 ? SG_STG1 : 2; }

struct SeqGridArgs {
  int d, d1, d2, nc, S;
  int ct;                      // columns per chain group (multiple of 8)
  int H;                       // chain groups per CTA column range
  int R;                       // row tiles per column range
  int tsmax;                   // largest T slice over tiles, doubles (rows x (KP + 4))
  unsigned long long* trace;   // optional start / end timestamps (CTA 0), debug only
  short r0[SG_MAXR], rows[SG_MAXR], kp[SG_MAXR], kt[SG_MAXR];
  const double* T;             // d x 2d row-major, columns [X ; Du ; Dw]
  const double* bias;          // d
  double* Z;                   // 2 x nc x 2d, permuted [X ; Dw ; Du]
  double* Xout;                // nc x d
  unsigned* cnt;               // one monotonic counter per chain group
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
__device__ __forceinline__ unsigned sg_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned sg_lds_acquire(unsigned addr) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sg_sts_release(unsigned addr, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ bool sg_mbar_test(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(  // try_wait suspends the thread for a while instead of spinning on the issue port
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void sg_bar_compute() {  // the 8 compute warps only
  asm volatile("bar.sync 1, %0;" ::"n"(SG_CTHREADS) : "memory");
}

// column k of the permuted contraction -> column of T's [X ; Du ; Dw] layout
__device__ __forceinline__ int sg_tcol(int k, int d, int d1, int d2) {
  if (k < d) return k;
  if (k < d + d2) return d + d1 + (k - d);  // Dw
  return d + (k - d - d2);                  // Du
}

// a poll that has not been answered after ~seconds means a lost CTA: fail loudly, never hang
constexpr unsigned SG_SPIN_LIMIT = 1u << 24;

template <int NT>
__global__ void __launch_bounds__(SG_THREADS, 1) seqgrid_kernel(const __grid_constant__ SeqGridArgs a) {
  const int cg = blockIdx.x / a.R, rt = blockIdx.x - (blockIdx.x / a.R) * a.R;
  const int r0 = a.r0[rt], RT = a.rows[rt], KP = a.kp[rt], KT = a.kt[rt];
  const int mt = RT >> 3;
  const int d = a.d, d1 = a.d1, d2 = a.d2, D2 = 2 * d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr int CT = NT * 8;
  constexpr int STG = sg_stages(NT);
  constexpr int ZS = SG_KCH + 4;                   // ring row stride (col-major chunk)
  constexpr int WRING = STG * CT * ZS;             // one warp's ring, doubles
  constexpr int WPART = SG_MT * NT * 64;           // one warp's partial tile (fragment order)
  const int SKO = KP + 4;                          // T slice row stride (conflict-free A)
  extern __shared__ __align__(16) double sm[];
  double* Ts = sm;                                 // RT x SKO
  double* ring = sm + a.tsmax;                     // warps x stages x CT x ZS
  double* part = ring + SG_CWARPS * WRING;         // warps x WPART
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(part + SG_CWARPS * WPART);
  const unsigned done_a = smem_u32(bars);          // done[i & 3]: sub-step i's stores issued
  const unsigned ready_a = smem_u32(bars + 4);     // sub-steps whose inputs are in L2

  // this CTA's chain groups and sub-step count
  const int ngrp = (a.nc + a.ct - 1) / a.ct;
  const int Hc = min(a.H, ngrp - cg * a.H);
  const int nsub = a.S * Hc;

  if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[8] = sg_timer();
  if (tid == 0) {
    // SG_MAXH barriers: sub-step i + SG_MAXH is admitted only after every CTA of the group
    // (this one included) has published i + SG_MAXH - Hc >= i, so a barrier never runs two
    // phases ahead of the publish warp
    for (int b = 0; b < SG_MAXH; ++b) mbar_init(done_a + 8 * b, SG_CWARPS);
    *reinterpret_cast<volatile unsigned*>(bars + 4) = (unsigned)Hc;  // step 0 needs no exchange
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // T slice -> smem in contraction order; rows past d and k past KT are zero.  One row per
  // warp pass, eight independent loads in flight per lane.
  if (((d1 | d2) & 1) == 0) {
    // even block sizes: the three segments of the permuted row start at even offsets, so the
    // slice goes global -> shared in 16-byte cp.async pieces with no register staging (a
    // scalar staged copy took 34 us of every launch at cfg2)
    const int np = KP >> 1;
    for (int idx = tid; idx < RT * np; idx += SG_THREADS) {
      const int r = idx / np, k = 2 * (idx - (idx / np) * np);
      const int gr = r0 + r;
      const bool ok = gr < d && k < KT;
      const double* src = ok ? a.T + (size_t)gr * D2 + sg_tcol(k, d, d1, d2) : a.T;
      sg_cp16(smem_u32(Ts + (size_t)r * SKO + k), src, ok ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  } else {
    for (int idx = tid; idx < RT * KP; idx += SG_THREADS) {
      const int r = idx / KP, k = idx - (idx / KP) * KP;
      const int gr = r0 + r;
      double v = 0.0;
      if (gr < d && k < KT) v = __ldg(a.T + (size_t)gr * D2 + sg_tcol(k, d, d1, d2));
      Ts[(size_t)r * SKO + k] = v;
    }
  }
  __syncthreads();
  if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[0] = sg_timer();

  if (warp == SG_CWARPS) {
    // ---- admit warp: sub-step (s, h) may start once every row tile has published (s-1, h)
    if (lane == 0) {
      for (int i = Hc; i < nsub; ++i) {  // step 0 of every group is admitted from the start
        const int s = i / Hc, h = i - (i / Hc) * Hc;
        const unsigned target = (unsigned)s * (unsigned)a.R;
        unsigned spins = 0;
        while (sg_ld_acquire(a.cnt + cg * a.H + h) < target)
          if (++spins > SG_SPIN_LIMIT) __trap();
        sg_sts_release(ready_a, (unsigned)(i + 1));
      }
    }
    return;
  }
  if (warp == SG_CWARPS + 1) {
    // ---- publish warp: the compute warps' stores (ordered by their mbarrier arrivals), then
    // the gpu-scope release increment of the group's counter
    if (lane == 0) {
      for (int i = 0; i < nsub; ++i) {
        const int h = i - (i / Hc) * Hc;
        const unsigned bar = done_a + 8 * (i & (SG_MAXH - 1));
        const unsigned par = (unsigned)((i / SG_MAXH) & 1);
        unsigned spins = 0;
        while (!sg_mbar_test(bar, par))
          if (++spins > SG_SPIN_LIMIT) __trap();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.cnt + cg * a.H + h)
                     : "memory");
      }
      if (a.trace && blockIdx.x == 0) a.trace[1] = sg_timer();
    }
    return;
  }

  // ---- compute warps --------------------------------------------------------------------
  // this warp's K slice, in whole chunks
  const int nch = KP / SG_KCH;
  const int cb = (warp * nch) / SG_WARPS, ce = ((warp + 1) * nch) / SG_WARPS;
  const int nw = ce - cb;
  double* myring = ring + (size_t)warp * WRING;
  double* mypart = part + (size_t)warp * WPART;
  const bool pf_ok = nw >= STG - 1;  // the next sub-step's prologue fits this one's tail

  // epilogue constants of this thread's outputs
  constexpr int OPT = (SG_MT * 8 * CT + SG_CTHREADS - 1) / SG_CTHREADS;
  double bo[OPT];
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int idx = tid + u * SG_CTHREADS;
    const int r = idx / CT;
    bo[u] = (idx < RT * CT && r0 + r < d) ? __ldg(a.bias + r0 + r) : 0.0;
  }

  auto zbase = [&](int i) {  // Z block read by sub-step i
    const int s = i / Hc, h = i - (i / Hc) * Hc;
    return a.Z + ((size_t)(s & 1) * a.nc + (size_t)(cg * a.H + h) * a.ct) * D2;
  };
  auto ncols = [&](int i) {
    const int h = i - (i / Hc) * Hc;
    return min(a.ct, a.nc - (cg * a.H + h) * a.ct);
  };
  auto load_chunk = [&](const double* Zp, int ncol, int ch, int slot) {
    double* dst = myring + (size_t)slot * CT * ZS;
    const int k0 = ch * SG_KCH;
    // CT columns x KCH k = CT x KCH/2 sixteen-byte pieces; 32 lanes
#pragma unroll
    for (int q0 = 0; q0 < CT * (SG_KCH / 2); q0 += 32) {
      const int q = lane + q0;
      const int col = q / (SG_KCH / 2), kk = (q % (SG_KCH / 2)) * 2;
      const int k = k0 + kk;
      const bool ok = col < ncol && k < KT;
      const double* src = ok ? Zp + (size_t)col * D2 + k : Zp;
      sg_cp16((unsigned)__cvta_generic_to_shared(dst + col * ZS + kk), src, ok ? 16 : 0);
    }
  };
  auto wait_ready = [&](int i) {  // blocks until sub-step i is admitted (warp-uniform)
    unsigned spins = 0;
    while (sg_lds_acquire(ready_a) <= (unsigned)i)
      if (++spins > SG_SPIN_LIMIT) __trap();
    __syncwarp();
  };

  int base = 0;       // ring slot of the sub-step's first chunk
  int issued = 0;     // chunks of the coming sub-step already in flight
  const bool tr = a.trace && blockIdx.x == 0 && tid == 0;
  unsigned long long t_wait = 0, t_main = 0, t_bar = 0, t_epi = 0, n_pf = 0, tq = 0;
  for (int i = 0; i < nsub; ++i) {
    if (tr) tq = sg_timer();
    const int s = i / Hc, h = i - (i / Hc) * Hc;
    const int c0 = (cg * a.H + h) * a.ct;
    const int ncol = min(a.ct, a.nc - c0);
    const double* Zp = zbase(i);
    if (issued == 0) {
      wait_ready(i);
      // prologue: STAGES-1 chunks in flight
#pragma unroll
      for (int j = 0; j < STG - 1; ++j) {
        if (j < nw) load_chunk(Zp, ncol, cb + j, (base + j) % STG);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
    } else if (tr) {
      ++n_pf;
    }
    if (tr) { const unsigned long long t = sg_timer(); t_wait += t - tq; tq = t; }
    // X_s of this thread's output rows (for D_{s+1}), fetched under the main loop
    double xo[OPT];
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int idx = tid + u * SG_CTHREADS;
      const int r = idx / CT, c = idx - (idx / CT) * CT;
      const bool ok = idx < RT * CT && r0 + r < d && c < ncol;
      xo[u] = ok ? __ldcg(Zp + (size_t)c * D2 + r0 + r) : 0.0;
    }
    // may the tail of this main loop stream the next sub-step's first chunks?
    bool pf = false;
    const double* Zn_in = Zp;
    int ncol_n = ncol;
    if (pf_ok && i + 1 < nsub) {
      Zn_in = zbase(i + 1);
      ncol_n = ncols(i + 1);
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
      for (int j = 0; j < nw; ++j) {
        const int ch = cb + j, slot = (base + j) % STG;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(STG - 2) : "memory");  // chunk j landed
        __syncwarp();  // ... for every lane; and the slot of chunk j-1 is no longer read
        const int jn = j + STG - 1;
        if (jn < nw) {
          load_chunk(Zp, ncol, cb + jn, (base + jn) % STG);
        } else if (pf_ok && i + 1 < nsub) {
          if (jn == nw) {  // first free slot of the tail: is the next sub-step admitted?
            const unsigned rdy = sg_lds_acquire(ready_a);
            pf = __all_sync(0xffffffffu, rdy > (unsigned)(i + 1));
          }
          if (pf) load_chunk(Zn_in, ncol_n, cb + (jn - nw), (base + jn) % STG);
        }
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
    issued = pf ? STG - 1 : 0;
    base = (base + nw) % STG;
    if (!pf) {  // nothing of the next sub-step is in flight: drain, all slots free
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      base = 0;
    }
    if (tr) { const unsigned long long t = sg_timer(); t_main += t - tq; tq = t; }
    // every compute thread has finished reading the previous sub-step's partials
    sg_bar_compute();
    if (tr) { const unsigned long long t = sg_timer(); t_bar += t - tq; tq = t; }
    // warp partial in fragment order ([m][n][lane][2]: one 16-byte store per fragment pair)
#pragma unroll
    for (int m = 0; m < SG_MT; ++m)
      if (m < mt)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          *reinterpret_cast<double2*>(mypart + ((m * NT + n) * 32 + lane) * 2) =
              make_double2(acc[m][n][0], acc[m][n][1]);
    sg_bar_compute();
    // fixed-order reduction over warps + epilogue, one (row, column) per thread
    double* Zn = a.Z + ((size_t)((s & 1) ^ 1) * a.nc + c0) * D2;
    const bool last = (s == a.S - 1);
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int idx = tid + u * SG_CTHREADS;
      const int r = idx / CT, c = idx - (idx / CT) * CT;
      const int gr = r0 + r;
      if (idx >= RT * CT || gr >= d || c >= ncol) continue;
      const int po = (((r >> 3) * NT + (c >> 3)) * 32 + (r & 7) * 4 + ((c & 7) >> 1)) * 2 + (c & 1);
      double v = 0.0;
      for (int w = 0; w < SG_WARPS; ++w) v += part[(size_t)w * WPART + po];
      v = __dadd_rn(v, bo[u]);
      const double dv = __dsub_rn(v, xo[u]);  // D_{s+1} = X_{s+1} - X_s
      double* zc = Zn + (size_t)c * D2;
      __stcg(zc + gr, v);
      __stcg(zc + (gr < d1 ? d + d2 + gr : d + (gr - d1)), dv);
      if (last) a.Xout[(size_t)(c0 + c) * d + gr] = v;
    }
    // hand the sub-step to the control warp: it publishes once all 8 warps have arrived
    __syncwarp();
    if (lane == 0) mbar_arrive(done_a + 8 * (i & (SG_MAXH - 1)));
    if (tr) { const unsigned long long t = sg_timer(); t_epi += t - tq; tq = t; }
  }
  if (tr) {
    a.trace[2] = t_wait;
    a.trace[3] = t_main;
    a.trace[4] = t_bar;
    a.trace[5] = t_epi;
    a.trace[6] = n_pf;
    a.trace[7] = (unsigned long long)nsub;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
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
  int ct = 0, H = 1, ncg = 0, R = 0;
  size_t tsmax = 0, smem = 0;
  long long cost = 0;
  short r0[SG_MAXR], rows[SG_MAXR], kp[SG_MAXR], kt[SG_MAXR];
};

static size_t sg_smem(size_t tsmax, int ct) {
  const int nt = ct / 8;
  const size_t ring = (size_t)sg_stages(nt) * ct * (SG_KCH + 4), part = (size_t)SG_MT * nt * 64;
  return sizeof(double) * (tsmax + (size_t)SG_CWARPS * (ring + part)) + 64;  // + barriers
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
  const size_t smem_cap = 227 * 1024;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sms = std::min(v, SG_MAXR);
  }
  best.ok = false;
  // experiment overrides (chain-group width / groups per CTA)
  static const int force_ct = getenv("PE_SEQGRID_CT") ? atoi(getenv("PE_SEQGRID_CT")) : 0;
  static const int force_h = getenv("PE_SEQGRID_H") ? atoi(getenv("PE_SEQGRID_H")) : 0;
  for (int ct = 8; ct <= 32; ct += 8) {
    if (force_ct && ct != force_ct) continue;
    const int ngrp = (nc + ct - 1) / ct;  // chain groups
    for (int H = 1; H <= SG_MAXH; ++H) {
      if (force_h && H != force_h) continue;
      if (H > ngrp) break;
      const int ncg = (ngrp + H - 1) / H;  // CTA column ranges
      const int R = sms / ncg;
      if (R < 1) continue;
      // smallest per-CTA DMMA cap (per chain group) that packs into R row tiles
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
      pl.H = H;
      pl.ncg = ncg;
      pl.cost = hi * H;  // DMMAs per CTA per step over its chain groups
      pl.smem = sg_smem(pl.tsmax, ct);
      pl.ok = true;
      // least work on the critical CTA; then more chain groups per CTA (their exchange
      // latencies overlap); then fewer CTAs
      if (!best.ok || pl.cost < best.cost || (pl.cost == best.cost && pl.H > best.H) ||
          (pl.cost == best.cost && pl.H == best.H && pl.ncg * pl.R < best.ncg * best.R))
        best = pl;
    }
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
  PE_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * pl.ncg * pl.H, st));
  SeqGridArgs a{};
  a.d = d;
  a.d1 = d1;
  a.d2 = d2;
  a.nc = nc;
  a.S = S;
  a.ct = pl.ct;
  a.H = pl.H;
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
    fprintf(stderr, "seqgrid plan: ct=%d H=%d ncg=%d R=%d ctas=%d smem=%zu cost=%lld\n", pl.ct,
            pl.H, pl.ncg, pl.R, pl.ncg * pl.R, pl.smem, pl.cost);
  const int grid = pl.ncg * pl.R;
  const int ntr = 9;
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
    fprintf(stderr, "seqgrid trace: T load %.1f us; %.3f us per step, total %.1f us (CTA 0, after the T load); "
            "per sub-step: admit wait %.3f main loop %.3f barrier %.3f epilogue %.3f us, "
            "prefetched %llu of %llu\n",
            (h[0] - h[8]) * 1e-3, (h[1] - h[0]) * 1e-3 / S, (h[1] - h[0]) * 1e-3, h[2] * 1e-3 / h[7], h[3] * 1e-3 / h[7],
            h[4] * 1e-3 / h[7], h[5] * 1e-3 / h[7], h[6], h[7]);
    cudaFree(a.trace);
  }
  return true;
}

}  // namespace pe
