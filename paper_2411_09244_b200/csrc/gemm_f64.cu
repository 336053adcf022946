// FP64 tensor-core (DMMA) batched GEMM with multi-segment K and fused epilogue.
//
// Every dense contraction of the hot path is one launch of this kernel:
//   * the sequential fine substep  X_{s+1} = T [X_s ; D_s] + c,  D_{s+1} = X_{s+1} - X_s
//     (stepping.py:122-147, composite operator built in setup.cu);
//   * the all-at-once right-hand side, time transforms, shifted complex applies and
//     the w-sweep (allatonce.py:112-158, 220-230).
// On sm_100a FP64 tensor work is warp-level DMMA only (tcgen05 has no f64 kind,
// SURVEY §0 F8): mma.sync.m8n8k4.f64 fed from shared memory, tiles staged with
// cp.async (LDGSTS) double buffering.

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <stdexcept>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "mbar.cuh"
#include "pe.h"
#include "pe_internal.h"

namespace pe {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Canonical k order of every libpe GEMM kernel: within each 16-deep k block, DMMA step q
// (q = 0..3) contracts k = q, q+4, q+8, q+12, lane t4 holding k = 4 t4 + q.  A lane's four
// fragments of one row are then one contiguous 32-byte run: two LDS.128 per fragment row
// per k block instead of four LDS.64, conflict-free for a row stride of 18 doubles (and for
// the 128-byte-swizzled TMA tiles).  Every kernel and variant uses this order, so results
// never depend on the tile choice (batch invariance).
template <int FM, int FN>
__device__ __forceinline__ void dmma_block16(const double* as, int sa, const double* bs, int sb,
                                             double (&acc)[FM][FN][2]) {
  double af[FM][4], bf[FN][4];
#pragma unroll
  for (int x = 0; x < FM; ++x) {
    const double2 u = *reinterpret_cast<const double2*>(as + x * 8 * sa);
    const double2 v = *reinterpret_cast<const double2*>(as + x * 8 * sa + 2);
    af[x][0] = u.x; af[x][1] = u.y; af[x][2] = v.x; af[x][3] = v.y;
  }
#pragma unroll
  for (int y = 0; y < FN; ++y) {
    const double2 u = *reinterpret_cast<const double2*>(bs + y * 8 * sb);
    const double2 v = *reinterpret_cast<const double2*>(bs + y * 8 * sb + 2);
    bf[y][0] = u.x; bf[y][1] = u.y; bf[y][2] = v.x; bf[y][3] = v.y;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int x = 0; x < FM; ++x)
#pragma unroll
      for (int y = 0; y < FN; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x][q], bf[y][q]);
}

// AK: A is k-contiguous (s1 == 1); BKC: B is k-contiguous (s0 == 1).
// Fused epilogue shared by both kernels: C = alpha acc + beta Cin + bias, D = C - Xp.
// Per fragment row the Cin / Xp loads are all issued before any store: C may alias Cin (the
// in-place recursion steps), which otherwise pins every load behind the previous store
// (one global-latency round trip per element).  Each thread reads only the elements it
// writes, so the hoisting is safe in place.
template <int FM, int FN>
__device__ __forceinline__ void gemm_epilogue(const GemmParams& p, int z1, int z2, int ibase,
                                              int jbase, const double (&acc)[FM][FN][2]) {
  if (p.nrm) {  // per-8-row-block column sums of squares; every lane takes part in the shuffles
    const int g = (threadIdx.x & 31) >> 2;
    const long long zc = (long long)(z1 * p.nb2 + z2) * p.N;
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int r0 = ibase - g + a * 8;  // first row of this fragment's 8-row block
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v = acc[a][b][h] * acc[a][b][h];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          const int gj = jbase + b * 8 + h;
          if (g == 0 && r0 < p.M && gj < p.N) p.nrm[(long long)(r0 >> 3) * p.nrm_ld + zc + gj] = v;
        }
    }
    return;
  }
  const long long cb = z1 * p.c_b1 + z2 * p.c_b2;
  double* C = p.C + cb;
  const double* Cin = p.Cin ? p.Cin + cb : nullptr;
  double* D = p.D ? p.D + cb : nullptr;
  const double* Xp = p.Xp ? p.Xp + cb : nullptr;
  const double* bias = p.bias ? p.bias + z1 * p.bias_b1 + z2 * p.bias_b2 : nullptr;
  const bool alpha1 = (p.alpha == 1.0), beta1 = (p.beta == 1.0);
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int gi = ibase + a * 8;
    if (gi >= p.M) continue;
    const long long ro = gi * p.c_i;
    // one prefetched operand per element: Cin when accumulating, else Xp for the D output
    // (no call site uses both; if one did, Xp is read late)
    const double* pf = Cin ? Cin : Xp;
    double pre[FN][2];
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = jbase + b * 8 + h;
        pre[b][h] = (pf && gj < p.N) ? pf[ro + gj * p.c_j] : 0.0;
      }
    const double bv = bias ? bias[gi] : 0.0;
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = jbase + b * 8 + h;
        if (gj >= p.N) continue;
        const long long off = ro + gj * p.c_j;
        double v = alpha1 ? acc[a][b][h] : __dmul_rn(p.alpha, acc[a][b][h]);
        if (Cin) v = __dadd_rn(v, beta1 ? pre[b][h] : __dmul_rn(p.beta, pre[b][h]));
        if (bias) v = __dadd_rn(v, bv);
        C[off] = v;
        if (D) D[off] = __dsub_rn(v, Cin ? Xp[off] : pre[b][h]);
      }
  }
}

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKC>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    gemm_f64_kernel(const __grid_constant__ GemmParams p) {
  pdl_enter();
  constexpr int WARPS_M = BM / WM;
  constexpr int NT = WARPS_M * (BN / WN) * 32;
  constexpr int FM = WM / 8, FN = WN / 8;
  static_assert(BK % 16 == 0, "k blocks of 16 (canonical k order)");
  constexpr int SK = BK + 2;  // row stride in doubles: conflict-free LDS.128 fragment runs
  __shared__ __align__(16) double As[2][BM * SK];
  __shared__ __align__(16) double Bs[2][BN * SK];

  const int z = blockIdx.z;
  const int z1 = z / p.nb2, z2 = z - (z / p.nb2) * p.nb2;
  const int i0 = blockIdx.y * BM;
  const int j0 = blockIdx.x * BN;

  int ntile = 0;
  int kt[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    kt[s] = (s < p.nseg) ? (p.seg[s].K + BK - 1) / BK : 0;
    ntile += kt[s];
  }

  auto load_tile = [&](int t, int buf) {
    int s = 0;
    while (t >= kt[s]) {
      t -= kt[s];
      ++s;
    }
    const GemmSeg& sg = p.seg[s];
    const int k0 = t * BK;
    const double* A = sg.A.p + z1 * sg.A.b1 + z2 * sg.A.b2;
    const double* B = sg.B.p + z1 * sg.B.b1 + z2 * sg.B.b2;
    const long long a0 = sg.A.s0, a1 = sg.A.s1, b0 = sg.B.s0, b1 = sg.B.s1;
    const int K = sg.K;
#pragma unroll 4
    for (int l = threadIdx.x; l < BM * BK; l += NT) {
      int ii, kk;
      if (AK) {
        ii = l / BK;
        kk = l - ii * BK;
      } else {
        kk = l / BM;
        ii = l - kk * BM;
      }
      const int gi = i0 + ii, gk = k0 + kk;
      const bool ok = (gi < p.M) && (gk < K);
      const double* src = ok ? (A + gi * a0 + gk * a1) : A;
      cp_async8(&As[buf][ii * SK + kk], src, ok);
    }
#pragma unroll 4
    for (int l = threadIdx.x; l < BN * BK; l += NT) {
      int jj, kk;
      if (BKC) {
        jj = l / BK;
        kk = l - jj * BK;
      } else {
        kk = l / BN;
        jj = l - kk * BN;
      }
      const int gj = j0 + jj, gk = k0 + kk;
      const bool ok = (gj < p.N) && (gk < K);
      const double* src = ok ? (B + gk * b0 + gj * b1) : B;
      cp_async8(&Bs[buf][jj * SK + kk], src, ok);
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int t0 = p.tri_upper ? min(ntile, i0 / BK) : 0;  // zero k-tiles of a triangular A
  if (ntile > t0) {
    load_tile(t0, t0 & 1);
    cp_async_commit();
    for (int t = t0; t < ntile; ++t) {
      const int buf = t & 1;
      if (t + 1 < ntile) {
        load_tile(t + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* as = &As[buf][(wm * WM + g) * SK + 4 * t4];
      const double* bs = &Bs[buf][(wn * WN + g) * SK + 4 * t4];
#pragma unroll
      for (int kb = 0; kb < BK; kb += 16) dmma_block16<FM, FN>(as + kb, SK, bs + kb, SK, acc);
      __syncthreads();
    }
  }

  // fused epilogue
  gemm_epilogue<FM, FN>(p, z1, z2, i0 + wm * WM + g, j0 + wn * WN + 2 * t4, acc);
}


// ----------------------------------------------------------------------------------------
// Fast path: A k-contiguous (row-major operators), B k-contiguous (BJC = false, the state /
// waveform columns) or j-contiguous (BJC = true, the time-transform operand).  16-byte
// cp.async.cg with per-thread precomputed offsets, a STAGES-deep pipeline with one CTA
// barrier per k-tile, 32x32 warp tiles (4x4 DMMA m8n8k4 accumulators per warp).  The k
// reduction order is the generic kernel's (k ascending in DMMA steps of 4 per segment), so
// both paths give bitwise identical results and may be mixed freely.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// Warp tile = (8 FM) x (8 FN) DMMA fragments, CTA = WGM x WGN warps.  Tile shapes that are
// not powers of two (64x72, 80x64) let the chooser fit the tile count to the 148 SMs.
template <int WGM, int WGN, int FM, int FN, int BK, int STAGES, bool BJC>
struct FastCfg {
  static constexpr int BM = WGM * 8 * FM;
  static constexpr int BN = WGN * 8 * FN;
  static constexpr int NT = WGM * WGN * 32;
  static constexpr int SA = BK + 2;
  static constexpr int SB = BJC ? (BN + 2) : (BK + 2);
  static constexpr int A_TILE = BM * SA;
  static constexpr int B_TILE = BJC ? BK * SB : BN * SB;
  static constexpr size_t SMEM = sizeof(double) * (size_t)STAGES * (A_TILE + B_TILE);
};

template <int WGM, int WGN, int FM, int FN, int BK, int STAGES, bool BJC, bool PRE = false>
__global__ void __launch_bounds__(WGM * WGN * 32)
    gemm_fast_kernel(const __grid_constant__ GemmParams p) {
  pdl_enter();
  using Cfg = FastCfg<WGM, WGN, FM, FN, BK, STAGES, BJC>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN;
  constexpr int NT = Cfg::NT, SA = Cfg::SA, SB = Cfg::SB;
  constexpr int WARPS_M = WGM;
  constexpr int WTM = 8 * FM, WTN = 8 * FN;
  extern __shared__ __align__(16) double smf[];
  double* As = smf;
  double* Bs = smf + STAGES * Cfg::A_TILE;

  const int zt = blockIdx.z;
  const int sp = zt % p.ksplit, z = zt / p.ksplit;
  const int z1 = z / p.nb2, z2 = z - (z / p.nb2) * p.nb2;
  // Grouped rasterisation for multi-wave grids: CTAs are dispatched in linear block order,
  // so walking `raster` row tiles down before stepping one column tile keeps a wave on a
  // near-square patch of C (its A and B panels are shared through L2 by the co-running
  // CTAs) instead of two full rows of tiles that re-stream all of B for every row tile.
  int ty = blockIdx.y, tx = blockIdx.x;
  if (p.raster > 1) {
    const int pid = blockIdx.y * gridDim.x + blockIdx.x, gsz = p.raster * gridDim.x;
    const int g = pid / gsz, first = g * p.raster, r = pid - g * gsz;
    const int gm = min(p.raster, (int)gridDim.y - first);
    ty = first + r % gm;
    tx = r / gm;
  }
  const int i0 = ty * BM, j0 = tx * BN;
  const int tid = threadIdx.x;

  int kt0 = 0, kt1 = 0, kt2 = 0;
  if (p.nseg > 0) kt0 = (p.seg[0].K + BK - 1) / BK;
  if (p.nseg > 1) kt1 = (p.seg[1].K + BK - 1) / BK;
  if (p.nseg > 2) kt2 = (p.seg[2].K + BK - 1) / BK;
  const int ktot = kt0 + kt1 + kt2;
  const int kper = (ktot + p.ksplit - 1) / p.ksplit;
  const int tskip = p.tri_upper ? min(ktot, i0 / BK) : 0;  // zero k-tiles of a triangular A
  const int tbeg = max(tskip, min(ktot, sp * kper));
  const int ntile = max(0, min(ktot, sp * kper + kper) - tbeg);  // this split's k-tiles

  // fixed per-thread chunk coordinates
  constexpr int ACPR = BK / 2;                 // 16-byte chunks per A row
  constexpr int AROWS = NT / ACPR;             // rows covered per pass
  constexpr int APASS = (BM + AROWS - 1) / AROWS;
  const int akc = tid % ACPR, ar = tid / ACPR;
  constexpr int BCPR = BJC ? BN / 2 : BK / 2;
  constexpr int BROWS = NT / BCPR;
  constexpr int BLEN = BJC ? BK : BN;
  constexpr int BPASS = (BLEN + BROWS - 1) / BROWS;
  const int bkc = tid % BCPR, br = tid / BCPR;
  const bool bload = br < BROWS;  // NT % BCPR threads left over (e.g. BN = 72) stay idle

  // Per-thread load descriptors of the segment being loaded: row pointers (batch offsets
  // and row strides folded in) and row-validity, computed once per segment instead of
  // once per k-tile; a k-tile then costs one add per 16-byte chunk.
  int lseg = -1, lK = 0;
  const double* arow[APASS];
  const double* brow[BPASS];
  bool aok[APASS], bok[BPASS];
  const double* Bbase = nullptr;
  long long bs0 = 0;
  auto set_seg = [&](int s) {
    const GemmSeg& sg = p.seg[s];
    const double* A = sg.A.p + z1 * sg.A.b1 + z2 * sg.A.b2;
    const double* B = sg.B.p + z1 * sg.B.b1 + z2 * sg.B.b2;
    lK = sg.K;
#pragma unroll
    for (int i = 0; i < APASS; ++i) {
      const int gi = i0 + ar + i * AROWS;
      aok[i] = gi < p.M;
      arow[i] = aok[i] ? A + (long long)gi * sg.A.s0 + 2 * akc : A;
    }
    if (!BJC) {
#pragma unroll
      for (int i = 0; i < BPASS; ++i) {
        const int gj = j0 + br + i * BROWS;
        bok[i] = gj < p.N;
        brow[i] = bok[i] ? B + (long long)gj * sg.B.s1 + 2 * bkc : B;
      }
    } else {
      Bbase = B;
      bs0 = sg.B.s0;
    }
    lseg = s;
  };
  auto load_tile_pre = [&](int t, int slot) {
    int s = 0, tt = t + tbeg;
    if (tt >= kt0) { tt -= kt0; s = 1; if (tt >= kt1) { tt -= kt1; s = 2; } }
    if (s != lseg) set_seg(s);
    const int k0 = tt * BK;
    double* as = As + slot * Cfg::A_TILE;
    double* bs = Bs + slot * Cfg::B_TILE;
    {
      const int kv = max(0, min(2, lK - (k0 + 2 * akc)));
#pragma unroll
      for (int i = 0; i < APASS; ++i) {
        const int r = ar + i * AROWS;
        if (ar >= AROWS || ((BM % AROWS) && r >= BM)) break;
        const int bytes = aok[i] ? 8 * kv : 0;
        cp_async16(as + r * SA + 2 * akc, bytes ? arow[i] + k0 : arow[i], bytes);
      }
    }
    if (!BJC) {
      const int kv = max(0, min(2, lK - (k0 + 2 * bkc)));
#pragma unroll
      for (int i = 0; i < BPASS; ++i) {
        const int r = br + i * BROWS;
        if (!bload || ((BLEN % BROWS) && r >= BLEN)) break;
        const int bytes = bok[i] ? 8 * kv : 0;
        cp_async16(bs + r * SB + 2 * bkc, bytes ? brow[i] + k0 : brow[i], bytes);
      }
    } else {
      const int jj = j0 + 2 * bkc;
      const int jv = max(0, min(2, p.N - jj));
#pragma unroll
      for (int i = 0; i < BPASS; ++i) {
        const int r = br + i * BROWS, gk = k0 + r;
        if (!bload || ((BLEN % BROWS) && r >= BLEN)) break;
        const int bytes = (gk < lK) ? 8 * jv : 0;
        const double* src = bytes ? Bbase + (long long)gk * bs0 + jj : Bbase;
        cp_async16(bs + r * SB + 2 * bkc, src, bytes);
      }
    }
  };

  auto load_tile_idx = [&](int t, int slot) {
    int s = 0, tt = t + tbeg;
    if (tt >= kt0) { tt -= kt0; s = 1; if (tt >= kt1) { tt -= kt1; s = 2; } }
    const GemmSeg& sg = p.seg[s];
    const int k0 = tt * BK, K = sg.K;
    const double* A = sg.A.p + z1 * sg.A.b1 + z2 * sg.A.b2;
    const double* B = sg.B.p + z1 * sg.B.b1 + z2 * sg.B.b2;
    double* as = As + slot * Cfg::A_TILE;
    double* bs = Bs + slot * Cfg::B_TILE;
    {
      const int kk = k0 + 2 * akc;
      const int kv = max(0, min(2, K - kk));
#pragma unroll
      for (int i = 0; i < APASS; ++i) {
        const int r = ar + i * AROWS, gi = i0 + r;
        if (ar >= AROWS || ((BM % AROWS) && r >= BM)) break;
        const int bytes = (gi < p.M) ? 8 * kv : 0;
        const double* src = bytes ? A + (long long)gi * sg.A.s0 + kk : A;
        cp_async16(as + r * SA + 2 * akc, src, bytes);
      }
    }
    if (!BJC) {
      const int kk = k0 + 2 * bkc;
      const int kv = max(0, min(2, K - kk));
#pragma unroll
      for (int i = 0; i < BPASS; ++i) {
        const int r = br + i * BROWS, gj = j0 + r;
        if (!bload || ((BLEN % BROWS) && r >= BLEN)) break;
        const int bytes = (gj < p.N) ? 8 * kv : 0;
        const double* src = bytes ? B + (long long)gj * sg.B.s1 + kk : B;
        cp_async16(bs + r * SB + 2 * bkc, src, bytes);
      }
    } else {
      const int jj = j0 + 2 * bkc;
      const int jv = max(0, min(2, p.N - jj));
#pragma unroll
      for (int i = 0; i < BPASS; ++i) {
        const int r = br + i * BROWS, gk = k0 + r;
        if (!bload || ((BLEN % BROWS) && r >= BLEN)) break;
        const int bytes = (gk < K) ? 8 * jv : 0;
        const double* src = bytes ? B + (long long)gk * sg.B.s0 + jj : B;
        cp_async16(bs + r * SB + 2 * bkc, src, bytes);
      }
    }
  };

  // Long-K products (cfg3: K = 8192) use the precomputed descriptors (rhs 32.1 -> 34.4
  // TF/s); short-K ones keep per-tile indexing, which needs fewer registers (102 vs 137 at
  // 64x72) and measured faster on the cfg2 shapes (66.8 vs 74.9 us)
  auto load_tile = [&](int t, int slot) {
    if constexpr (PRE && !BJC)
      load_tile_pre(t, slot);
    else
      load_tile_idx(t, slot);
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < ntile) load_tile(st, st);
    cp_async_commit();
  }
  for (int t = 0; t < ntile; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (t + STAGES - 1 < ntile) load_tile(t + STAGES - 1, (t + STAGES - 1) % STAGES);
    cp_async_commit();
    const int slot = t % STAGES;
    const double* as = As + slot * Cfg::A_TILE + (wm * WTM + g) * SA + 4 * t4;
    if (!BJC) {
      const double* bs = Bs + slot * Cfg::B_TILE + (wn * WTN + g) * SB + 4 * t4;
#pragma unroll
      for (int kb = 0; kb < BK; kb += 16) dmma_block16<FM, FN>(as + kb, SA, bs + kb, SB, acc);
    } else {  // B stored [k][j]: the lane's k run is strided; same canonical k order
      const double* bs = Bs + slot * Cfg::B_TILE + (4 * t4) * SB + wn * WTN + g;
#pragma unroll
      for (int kb = 0; kb < BK; kb += 16) {
        double af[FM][4], bf[FN][4];
#pragma unroll
        for (int x = 0; x < FM; ++x) {
          const double2 u = *reinterpret_cast<const double2*>(as + kb + x * 8 * SA);
          const double2 v = *reinterpret_cast<const double2*>(as + kb + x * 8 * SA + 2);
          af[x][0] = u.x; af[x][1] = u.y; af[x][2] = v.x; af[x][3] = v.y;
        }
#pragma unroll
        for (int y = 0; y < FN; ++y)
#pragma unroll
          for (int q = 0; q < 4; ++q) bf[y][q] = bs[(kb + q) * SB + y * 8];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int x = 0; x < FM; ++x)
#pragma unroll
            for (int y = 0; y < FN; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x][q], bf[y][q]);
      }
    }
  }
  cp_async_wait<0>();

  if (p.ksplit > 1) {  // raw partial tile -> ws[sp][z][j][i]; splitk_reduce_kernel finishes
    const int batch = p.nb1 * p.nb2;
    const size_t plane = (size_t)batch * p.M * p.N;
    double* W = p.ws + (size_t)sp * plane + (size_t)z * p.M * p.N;
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int gi = i0 + wm * WTM + a * 8 + g;
      if (gi >= p.M) continue;
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gj = j0 + wn * WTN + b * 8 + 2 * t4 + h;
          if (gj < p.N) W[(size_t)gj * p.M + gi] = acc[a][b][h];
        }
    }
    return;
  }

  gemm_epilogue<FM, FN>(p, z1, z2, i0 + wm * WTM + g, j0 + wn * WTN + 2 * t4, acc);
}

// Split-K reduction: C = alpha * sum_sp ws[sp] (splits in order) + epilogue.
__global__ void splitk_reduce_kernel(const __grid_constant__ GemmParams p) {
  pdl_enter();
  const int batch = p.nb1 * p.nb2;
  const long long per = (long long)p.M * p.N;
  const long long total = per * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int z = (int)(t / per);
    const long long r = t - z * per;
    const int gj = (int)(r / p.M), gi = (int)(r - (long long)gj * p.M);
    double v = 0.0;
    for (int sp = 0; sp < p.ksplit; ++sp) v += p.ws[(size_t)sp * total + t];
    const int z1 = z / p.nb2, z2 = z - (z / p.nb2) * p.nb2;
    const long long cb = z1 * p.c_b1 + z2 * p.c_b2;
    const long long off = cb + gi * p.c_i + gj * p.c_j;
    if (p.alpha != 1.0) v = __dmul_rn(p.alpha, v);
    if (p.Cin) v = __dadd_rn(v, p.beta == 1.0 ? p.Cin[off] : __dmul_rn(p.beta, p.Cin[off]));
    if (p.bias) v = __dadd_rn(v, p.bias[z1 * p.bias_b1 + z2 * p.bias_b2 + gi]);
    p.C[off] = v;
    if (p.D) p.D[off] = __dsub_rn(v, p.Xp[off]);
  }
}

template <int WGM, int WGN, int FM, int FN, int BK, int STAGES, bool BJC, bool PRE = false>
static int fast_occupancy() {
  static int occ = -1;
  if (occ < 0) {
    using Cfg = FastCfg<WGM, WGN, FM, FN, BK, STAGES, BJC>;
    auto kern = gemm_fast_kernel<WGM, WGN, FM, FN, BK, STAGES, BJC, PRE>;
    PE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Cfg::SMEM));
    int n = 0;
    PE_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, Cfg::NT, Cfg::SMEM));
    occ = n;
  }
  return occ;
}

template <int WGM, int WGN, int FM, int FN, int BK, int STAGES, bool BJC, bool PRE = false>
static void launch_fast(const GemmParams& p, cudaStream_t st) {
  using Cfg = FastCfg<WGM, WGN, FM, FN, BK, STAGES, BJC>;
  const int occ = fast_occupancy<WGM, WGN, FM, FN, BK, STAGES, BJC, PRE>();
  dim3 grid((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM, p.nb1 * p.nb2 * p.ksplit);
  GemmParams q = p;
  // more than two waves per batch slice and enough row tiles to group
  static const int raster_env = std::getenv("PE_GEMM_RASTER") ? std::atoi(std::getenv("PE_GEMM_RASTER")) : 16;
  if (raster_env > 1 && grid.y >= 4 && (long long)grid.x * grid.y > 2LL * 148 * std::max(1, occ))
    q.raster = std::min<int>(raster_env, grid.y);
  launch_k(gemm_fast_kernel<WGM, WGN, FM, FN, BK, STAGES, BJC, PRE>, grid, dim3(Cfg::NT), Cfg::SMEM, st, q);
  ++g_launches;
}

static bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

// Fast-path eligibility: 16-byte chunks along the contiguous dimension of A and B.
static int fast_layout(const GemmParams& p) {
  if (p.nseg == 0) return -1;
  int bjc = -1;
  for (int s = 0; s < p.nseg; ++s) {
    const Operand& A = p.seg[s].A;
    const Operand& B = p.seg[s].B;
    if (A.s1 != 1 || (A.s0 & 1) || (A.b1 & 1) || (A.b2 & 1) || !aligned16(A.p)) return -1;
    int lay;
    if (B.s0 == 1 && !(B.s1 & 1)) lay = 0;
    else if (B.s1 == 1 && !(B.s0 & 1)) lay = 1;
    else return -1;
    if ((B.b1 & 1) || (B.b2 & 1) || !aligned16(B.p)) return -1;
    if (bjc >= 0 && lay != bjc) return -1;
    bjc = lay;
  }
  return bjc;
}

// Fast-path variants: id, warps (M, N), fragments per warp (M, N), BK, stages, auto.
// Every variant accumulates k in the same order, so the choice never changes a result bit.
// auto = 1: considered by the cost model; 0: reachable through PE_GEMM_VARIANT only
// (measured slower on every hot-path shape, tools/gemm_bench.py).
#define PE_FAST_VARIANTS(X)   \
  X(0, 2, 2, 4, 4, 32, 3, 0)  \
  X(1, 2, 2, 4, 4, 16, 3, 0)  \
  X(2, 4, 2, 4, 4, 16, 3, 0)  \
  X(3, 4, 1, 4, 4, 32, 3, 0)  \
  X(5, 2, 2, 4, 4, 16, 2, 1)  \
  X(6, 2, 2, 4, 4, 32, 2, 0)  \
  X(7, 2, 1, 4, 4, 16, 2, 1)  \
  X(8, 2, 3, 4, 3, 16, 2, 1)  \
  X(9, 2, 2, 5, 4, 16, 2, 1)  \
  X(10, 1, 2, 5, 4, 16, 2, 1) \
  X(11, 2, 3, 4, 3, 16, 3, 0) \
  X(12, 4, 1, 5, 4, 16, 2, 1) \
  X(13, 3, 1, 5, 4, 16, 2, 0) \
  X(14, 2, 3, 4, 3, 32, 2, 0) \
  X(15, 2, 3, 4, 3, 32, 3, 0) \
  X(16, 4, 3, 4, 3, 16, 3, 0) \
  X(17, 2, 3, 5, 3, 16, 2, 0) \
  X(18, 2, 3, 5, 3, 32, 2, 0) \
  X(19, 2, 2, 5, 4, 32, 2, 0)

static constexpr int kMaxVariant = 20;

// Wave-quantised cost: CTAs are spread round-robin over the 148 SMs and the SM with the
// most tiles finishes last; its work is max_tiles x tile area (padding included).
// 2-warp CTAs sustain ~20 % less DMMA issue per SM (measured: 64x32 vs 64x64).
template <int WGM, int WGN, int FM, int FN, int BK, int STAGES, bool BJC>
static double fast_cost(const GemmParams& p) {
  using Cfg = FastCfg<WGM, WGN, FM, FN, BK, STAGES, BJC>;
  const int occ = fast_occupancy<WGM, WGN, FM, FN, BK, STAGES, BJC>();
  if (occ <= 0) return 1e300;
  const double ctas = (double)((p.M + Cfg::BM - 1) / Cfg::BM) * ((p.N + Cfg::BN - 1) / Cfg::BN) *
                      p.nb1 * p.nb2;
  const double per_sm = std::ceil(ctas / 148.0);
  const double eff = (WGM * WGN <= 2) ? 0.8 : 1.0;
  return per_sm * Cfg::BM * Cfg::BN / eff;
}

template <bool BJC>
static void launch_variant(int id, const GemmParams& p, cudaStream_t st, bool pre = false) {
  switch (id) {
#define PE_X(ID, WGM, WGN, FM, FN, BK, ST, AUTO)                              \
  case ID:                                                                    \
    if (!BJC && pre)                                                          \
      launch_fast<WGM, WGN, FM, FN, BK, ST, BJC, !BJC>(p, st);                \
    else                                                                      \
      launch_fast<WGM, WGN, FM, FN, BK, ST, BJC>(p, st);                      \
    return;
    PE_FAST_VARIANTS(PE_X)
#undef PE_X
    default:
      launch_fast<2, 2, 4, 4, 16, 2, BJC>(p, st);
  }
}

template <bool BJC>
static int choose_variant(const GemmParams& p) {
  int best = 5;
  double bc = 1e300;
#define PE_X(ID, WGM, WGN, FM, FN, BK, ST, AUTO)                     \
  if (AUTO) {                                                        \
    const double c = fast_cost<WGM, WGN, FM, FN, BK, ST, BJC>(p);   \
    if (c < bc * 0.97) {                                             \
      bc = c;                                                        \
      best = ID;                                                     \
    }                                                                \
  }
  PE_FAST_VARIANTS(PE_X)
#undef PE_X
  return best;
}

template <int BM, int BN, int BK, int WM, int WN>
static void launch_cfg(const GemmParams& p, bool ak, bool bk, cudaStream_t st) {
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.nb1 * p.nb2);
  dim3 block((BM / WM) * (BN / WN) * 32);
  if (ak && bk)
    launch_k(gemm_f64_kernel<BM, BN, BK, WM, WN, true, true>, grid, block, 0, st, p);
  else if (ak && !bk)
    launch_k(gemm_f64_kernel<BM, BN, BK, WM, WN, true, false>, grid, block, 0, st, p);
  else if (!ak && bk)
    launch_k(gemm_f64_kernel<BM, BN, BK, WM, WN, false, true>, grid, block, 0, st, p);
  else
    launch_k(gemm_f64_kernel<BM, BN, BK, WM, WN, false, false>, grid, block, 0, st, p);
  ++g_launches;
}

double gemm_flops(const GemmParams& p) {
  double k = 0;
  for (int s = 0; s < p.nseg; ++s) k += p.seg[s].K;
  double mk = p.M * k;
  if (p.tri_upper && p.nseg == 1) {  // nonzeros of an upper-triangular M x K operator
    const double m = std::min<double>(p.M, k);
    mk = m * k - m * (m - 1) / 2;
  }
  return 2.0 * mk * (double)p.N * p.nb1 * p.nb2;
}

// ----------------------------------------------------------------------------------------
// TMA path (both operands k-contiguous): one producer warp streams the A and B k-tiles of
// every segment with cp.async.bulk.tensor into a STAGES-deep ring of 128-byte-swizzled
// shared tiles, signalling a "full" mbarrier per stage by transaction bytes; the DMMA
// warps wait on it, consume the 16-deep k-tile and release the stage through an "empty"
// mbarrier.  No CTA barrier and no per-thread address arithmetic in the main loop.  Tiles
// are zero-filled out of bounds, the k order is the cp.async kernels' (segment by segment,
// k ascending in DMMA steps of 4), so every path gives the same bits.
struct alignas(64) TmaArgs {
  CUtensorMap ta[3];
  CUtensorMap tb[3];
  GemmParams p;
  int za[3][2], zb[3][2];  // per segment: use (z1, z2) as TMA batch coordinates (0: shared)
};

template <int WGM, int WGN, int FM, int FN, int STAGES>
struct TmaCfg {
  static constexpr int BM = WGM * 8 * FM, BN = WGN * 8 * FN, BK = 16;
  static constexpr int NCW = WGM * WGN;         // DMMA (consumer) warps
  static constexpr int NT = (NCW + 1) * 32;     // + one producer warp
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 2 * STAGES * 8;
};

// byte offset of element (r, k) (k < 16) in a 128B-swizzled [rows][16 doubles] tile
__device__ __forceinline__ unsigned swz(int r, int k) {
  return (unsigned)(r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3));
}

template <int WGM, int WGN, int FM, int FN, int STAGES>
__global__ void __launch_bounds__((WGM * WGN + 1) * 32)
    gemm_tma_kernel(const __grid_constant__ TmaArgs a) {
  using Cfg = TmaCfg<WGM, WGN, FM, FN, STAGES>;
  constexpr int NCW = Cfg::NCW;
  constexpr int WTM = 8 * FM, WTN = 8 * FN;
  extern __shared__ unsigned char smraw[];
  const unsigned sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const unsigned char* sgen = smraw + (sbase - smem_u32(smraw));
  const unsigned bar_full = sbase + STAGES * Cfg::STAGE;
  const unsigned bar_empty = bar_full + STAGES * 8;
  const GemmParams& p = a.p;
  const int z = blockIdx.z;
  const int z1 = z / p.nb2, z2 = z - (z / p.nb2) * p.nb2;
  int ty = blockIdx.y, tx = blockIdx.x;
  if (p.raster > 1) {  // grouped rasterisation, as gemm_fast_kernel
    const int pid = blockIdx.y * gridDim.x + blockIdx.x, gsz = p.raster * gridDim.x;
    const int gq = pid / gsz, first = gq * p.raster, r = pid - gq * gsz;
    const int gm = min(p.raster, (int)gridDim.y - first);
    ty = first + r % gm;
    tx = r / gm;
  }
  const int i0 = ty * Cfg::BM, j0 = tx * Cfg::BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int kt[3] = {0, 0, 0};
  for (int s = 0; s < p.nseg; ++s) kt[s] = (p.seg[s].K + 15) / 16;
  const int ktot = kt[0] + kt[1] + kt[2];
  const int tskip = p.tri_upper ? min(ktot, i0 / 16) : 0;
  const int ntile = ktot - tskip;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();

  if (warp == NCW) {  // producer
    if (lane == 0) {
      for (int t = 0; t < ntile; ++t) {
        const int st = t % STAGES;
        if (t >= STAGES) mbar_wait_cta(bar_empty + 8 * st, ((t / STAGES) - 1) & 1);
        int g = t + tskip, s = 0;
        if (g >= kt[0]) { g -= kt[0]; s = 1; if (g >= kt[1]) { g -= kt[1]; s = 2; } }
        const unsigned full = bar_full + 8 * st;
        mbar_expect_tx(full, Cfg::STAGE);
        const unsigned dA = sbase + st * Cfg::STAGE;
        tma_load_4d(dA, &a.ta[s], g * 16, i0, a.za[s][1] ? z2 : 0, a.za[s][0] ? z1 : 0, full);
        tma_load_4d(dA + Cfg::A_BYTES, &a.tb[s], g * 16, j0, a.zb[s][1] ? z2 : 0,
                    a.zb[s][0] ? z1 : 0, full);
      }
    }
    return;
  }

  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp % WGM, wn = warp / WGM;
  // swizzled offsets of the lane's k run (row g, k = 4 t4 .. 4 t4 + 3): two 16-byte chunks
  const unsigned ko0 = swz(g, 4 * t4), ko1 = swz(g, 4 * t4 + 2);
  double acc[FM][FN][2];
#pragma unroll
  for (int x = 0; x < FM; ++x)
#pragma unroll
    for (int y = 0; y < FN; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

  for (int t = 0; t < ntile; ++t) {
    const int st = t % STAGES;
    mbar_wait_cta(bar_full + 8 * st, (t / STAGES) & 1);
    const unsigned char* sa = sgen + st * Cfg::STAGE + (wm * WTM) * 128;
    const unsigned char* sb = sgen + st * Cfg::STAGE + Cfg::A_BYTES + (wn * WTN) * 128;
    double af[FM][4], bf[FN][4];
#pragma unroll
    for (int x = 0; x < FM; ++x) {
      const double2 u = *reinterpret_cast<const double2*>(sa + x * 8 * 128 + ko0);
      const double2 v = *reinterpret_cast<const double2*>(sa + x * 8 * 128 + ko1);
      af[x][0] = u.x; af[x][1] = u.y; af[x][2] = v.x; af[x][3] = v.y;
    }
#pragma unroll
    for (int y = 0; y < FN; ++y) {
      const double2 u = *reinterpret_cast<const double2*>(sb + y * 8 * 128 + ko0);
      const double2 v = *reinterpret_cast<const double2*>(sb + y * 8 * 128 + ko1);
      bf[y][0] = u.x; bf[y][1] = u.y; bf[y][2] = v.x; bf[y][3] = v.y;
    }
    // the fragments are in registers: hand the stage back before the DMMAs
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * st);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int x = 0; x < FM; ++x)
#pragma unroll
        for (int y = 0; y < FN; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x][q], bf[y][q]);
  }
  gemm_epilogue<FM, FN>(p, z1, z2, i0 + wm * WTM + g, j0 + wn * WTN + 2 * t4, acc);
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    PE_CUDA_CHECK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000,
                                                   cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      throw Error{PE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 4-D map {k, row, z2, z1} of a k-contiguous FP64 operand; a zero batch stride collapses
// that level (extent 1, coordinate 0).  Box = 16 k x box_rows rows, 128-byte swizzle.
static void encode_operand(CUtensorMap* m, int use[2], const double* base, int K, int rows,
                           long long row_stride, long long b1, int n1, long long b2, int n2,
                           int box_rows) {
  const cuuint64_t span = (cuuint64_t)row_stride * rows * 8;
  cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)(b2 ? n2 : 1),
                        (cuuint64_t)(b1 ? n1 : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)row_stride * 8, (cuuint64_t)(b2 ? b2 * 8 : ((span + 15) & ~15ull)),
                           (cuuint64_t)(b1 ? b1 * 8 : ((span + 15) & ~15ull))};
  cuuint32_t box[4] = {16, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  use[0] = b1 != 0;
  use[1] = b2 != 0;
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                          const_cast<double*>(base), dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error{PE_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
}

// TMA eligibility: every segment k-contiguous in both operands, 16-byte aligned bases,
// even (16-byte) row and batch strides, no split-K.
static bool tma_ok(const GemmParams& p) {
  static const bool off = getenv("PE_GEMM_NO_TMA") != nullptr;
  if (off || p.nseg == 0) return false;
  for (int s = 0; s < p.nseg; ++s) {
    const Operand& A = p.seg[s].A;
    const Operand& B = p.seg[s].B;
    if (A.s1 != 1 || B.s0 != 1) return false;
    if ((A.s0 & 1) || (B.s1 & 1) || (A.b1 & 1) || (A.b2 & 1) || (B.b1 & 1) || (B.b2 & 1)) return false;
    if (A.s0 <= 0 || B.s1 <= 0 || A.b1 < 0 || A.b2 < 0 || B.b1 < 0 || B.b2 < 0) return false;
    if (!aligned16(A.p) || !aligned16(B.p) || p.seg[s].K <= 0) return false;
  }
  return true;
}

template <int WGM, int WGN, int FM, int FN, int STAGES>
static void launch_tma(const GemmParams& p, cudaStream_t st) {
  using Cfg = TmaCfg<WGM, WGN, FM, FN, STAGES>;
  static bool attr = false;
  auto kern = gemm_tma_kernel<WGM, WGN, FM, FN, STAGES>;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr = true;
  }
  TmaArgs a;
  memset(static_cast<void*>(&a), 0, sizeof(a));
  a.p = p;
  a.p.ksplit = 1;
  for (int s = 0; s < p.nseg; ++s) {
    const GemmSeg& g = p.seg[s];
    encode_operand(&a.ta[s], a.za[s], g.A.p, g.K, p.M, g.A.s0, g.A.b1, p.nb1, g.A.b2, p.nb2, Cfg::BM);
    encode_operand(&a.tb[s], a.zb[s], g.B.p, g.K, p.N, g.B.s1, g.B.b1, p.nb1, g.B.b2, p.nb2, Cfg::BN);
  }
  dim3 grid((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM, p.nb1 * p.nb2);
  static const int raster_env = std::getenv("PE_GEMM_RASTER") ? std::atoi(std::getenv("PE_GEMM_RASTER")) : 16;
  if (raster_env > 1 && grid.y >= 4 && (long long)grid.x * grid.y > 6LL * 148)
    a.p.raster = std::min<int>(raster_env, grid.y);
  launch_k(kern, grid, dim3(Cfg::NT), Cfg::SMEM, st, a);
  ++g_launches;
}

// TMA variants: id, consumer warps (M, N), fragments per warp (M, N), stages.
#define PE_TMA_VARIANTS(X) \
  X(0, 2, 3, 4, 3, 4)      \
  X(1, 2, 2, 4, 4, 4)      \
  X(2, 4, 2, 4, 4, 3)      \
  X(3, 2, 2, 5, 4, 4)      \
  X(4, 1, 2, 4, 4, 4)      \
  X(5, 2, 4, 4, 4, 3)      \
  X(6, 4, 1, 4, 4, 4)      \
  X(7, 3, 1, 5, 4, 4)      \
  X(8, 2, 1, 5, 4, 4)      \
  X(9, 5, 1, 4, 4, 4)      \
  X(10, 5, 1, 4, 4, 3)

template <int WGM, int WGN, int FM, int FN, int STAGES>
static double tma_cost(const GemmParams& p) {
  using Cfg = TmaCfg<WGM, WGN, FM, FN, STAGES>;
  const double ctas = (double)((p.M + Cfg::BM - 1) / Cfg::BM) * ((p.N + Cfg::BN - 1) / Cfg::BN) *
                      p.nb1 * p.nb2;
  const double per_sm = std::ceil(ctas / 148.0);
  // fewer DMMA warps per CTA sustain less issue (measured at cfg4, 600 x 32 x 1200 x 32:
  // 128x32 / 4 warps 7.26 ms per iteration, 120x32 / 3 warps 8.57, 80x32 / 2 warps 8.82)
  const double eff = (Cfg::NCW <= 2) ? 0.6 : (Cfg::NCW == 3 ? 0.8 : 1.0);
  return per_sm * Cfg::BM * Cfg::BN / eff;
}

static void launch_tma_best(const GemmParams& p, cudaStream_t st) {
  static const int forced = getenv("PE_TMA_VARIANT") ? atoi(getenv("PE_TMA_VARIANT")) : -1;
  int best = 0;
  double bc = 1e300;
#define PE_X(ID, WGM, WGN, FM, FN, ST)                         \
  {                                                            \
    const double c = tma_cost<WGM, WGN, FM, FN, ST>(p);        \
    if (c < bc * 0.97) {                                       \
      bc = c;                                                  \
      best = ID;                                               \
    }                                                          \
  }
  PE_TMA_VARIANTS(PE_X)
#undef PE_X
  if (forced >= 0) best = forced;
  switch (best) {
#define PE_X(ID, WGM, WGN, FM, FN, ST) \
  case ID:                             \
    launch_tma<WGM, WGN, FM, FN, ST>(p, st); \
    return;
    PE_TMA_VARIANTS(PE_X)
#undef PE_X
    default:
      launch_tma<2, 3, 4, 3, 4>(p, st);
  }
}

// ----------------------------------------------------------------------------------------
// Row-balanced persistent variant for batched skinny products (the ensemble fine step, cfg4:
// E members x (d x 2d)(2d x nc), nc <= 32).  The E * M rows are split in 8-row blocks into
// one contiguous range per SM (max/mean 1.02 at cfg4, where 160-row tiles leave 40 SMs
// with half the work of the others).  A range covers at most two members (a "part" each);
// both parts run through ONE k-loop: every consumer warp owns 4 consecutive m-blocks
// (32 rows) of one part, and each stage holds the part's A blocks plus one B tile per part.
// Rows below `zero_rows` have an exact-zero k-range [zero_k0, zero_k1) of the second
// segment (segment-local k; the composite step's u x Du block): a warp whose four blocks
// all lie below it neither loads nor multiplies those k-tiles.  One producer warp issues
// one 8-row 128B-swizzled TMA box per loaded m-block and one box per B tile.  Same
// canonical k order and epilogue as the other kernels, so a result differs from theirs only
// by the omitted +0 terms.
#ifndef RB_WARPS_N
#define RB_WARPS_N 11
#endif
// ring depth: measured at cfg4 with the chained kernel (GEMM ms per iteration) 4 stages 3.30,
// 3 stages 3.34, 2 stages 3.38 -- the consumers are not waiting for HBM latency; a stage is
// released by ALL warps, so the warps of a CTA move through the k-tiles in step
#ifndef RB_STAGES_N
#define RB_STAGES_N 4
#endif
constexpr int RB_WARPS = RB_WARPS_N, RB_FM = 4, RB_FN = 4, RB_STAGES = RB_STAGES_N;  // + the producer warp
constexpr int RB_MAXB = 40;  // m-blocks per CTA range: ceil(a/4) + ceil(b/4) <= 11
constexpr int RB_A_BYTES = RB_MAXB * 1024, RB_B_BYTES = 8 * RB_FN * 128;
constexpr int RB_STAGE = RB_A_BYTES + 2 * RB_B_BYTES;
constexpr size_t RB_SMEM = (size_t)RB_STAGES * RB_STAGE + 1024 + 2 * RB_STAGES * 8;

struct alignas(64) RowBalArgs {
  CUtensorMap ta[2];  // A segment maps {K_s, E * M} (box 16 x 8 rows)
  CUtensorMap ta4[2];  // the same with 32-row boxes (a full warp's four blocks, one TMA)
  CUtensorMap tb[2];  // B segment maps {K_s, E * N} (box 16 x 8 FN rows)
  GemmParams p;
  int blocks;         // E * M / 8
  int zero_rows, zk0, zk1;
  // work-weighted split: a member-local block below zero_rows / 8 weighs wu k-tiles (its
  // zero k-tiles are skipped), any other block ww; CTA c starts at weight W c / grid
  int wu, ww, zrb;
};

// CTA range -> up to two parts (member, first member-local block, block count) and the
// warp layout: part 0 takes warps [0, w0), part 1 [w0, w0 + w1), 4 blocks per warp.
struct RbPlan {
  int e[2], sb[2], nb[2], w0, nw;
};
// first block whose cumulative weight reaches w (blocks in member-major order)
// geometry of a row-balanced split: M rows per member, `blocks` 8-row blocks in all, the
// first zrb blocks of a member weigh wu k-tiles, the others ww
struct RbGeom {
  int M, blocks, zrb, wu, ww;
};
template <class Args>
__device__ __forceinline__ RbGeom rb_geom(const Args& a) {
  return RbGeom{a.p.M, a.blocks, a.zrb, a.wu, a.ww};
}
// first block whose cumulative weight reaches w (blocks in member-major order)
__device__ __forceinline__ long long rb_block_at(const RbGeom& a, long long w) {
  const int mb = a.M / 8;
  const long long wm = (long long)a.zrb * a.wu + (long long)(mb - a.zrb) * a.ww;
  const long long e = w / wm;
  long long r = w - e * wm;
  long long b;
  if (r < (long long)a.zrb * a.wu)
    b = (r + a.wu - 1) / a.wu;
  else
    b = a.zrb + (r - (long long)a.zrb * a.wu + a.ww - 1) / a.ww;
  return e * mb + b;
}
// block range [b0, b1) of CTA c
__device__ __forceinline__ void rb_range(const RbGeom& a, int c, long long& b0, long long& b1) {
  const int mb = a.M / 8;
  const long long E = a.blocks / mb;
  const long long W = E * ((long long)a.zrb * a.wu + (long long)(mb - a.zrb) * a.ww);
  b0 = c == 0 ? 0 : rb_block_at(a, W * c / gridDim.x);
  b1 = c + 1 == (int)gridDim.x ? a.blocks : rb_block_at(a, W * (c + 1) / gridDim.x);
}
__device__ __forceinline__ RbPlan rb_plan(const RbGeom& a) {
  const int mb = a.M / 8;
  long long b0, b1;
  rb_range(a, (int)blockIdx.x, b0, b1);
  RbPlan r;
  r.e[0] = (int)(b0 / mb);
  r.sb[0] = (int)(b0 - (long long)r.e[0] * mb);
  const long long end0 = (long long)(r.e[0] + 1) * mb;
  r.nb[0] = (int)((b1 < end0 ? b1 : end0) - b0);
  r.e[1] = r.e[0] + 1;
  r.sb[1] = 0;
  r.nb[1] = b1 > end0 ? (int)(b1 - end0) : 0;
  r.w0 = (r.nb[0] + RB_FM - 1) / RB_FM;
  r.nw = r.w0 + (r.nb[1] + RB_FM - 1) / RB_FM;
  return r;
}

__global__ void __launch_bounds__((RB_WARPS + 1) * 32, 1)
    gemm_rowbal_kernel(const __grid_constant__ RowBalArgs a) {
  extern __shared__ unsigned char smraw[];
  const unsigned sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const unsigned char* sgen = smraw + (sbase - smem_u32(smraw));
  const unsigned bar_full = sbase + RB_STAGES * RB_STAGE;
  const unsigned bar_empty = bar_full + RB_STAGES * 8;
  const GemmParams& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RbPlan pl = rb_plan(rb_geom(a));
  const int kt0 = (p.seg[0].K + 15) / 16, kt1 = p.nseg > 1 ? (p.seg[1].K + 15) / 16 : 0;
  const int ktot = kt0 + kt1;
  // k-tiles of the second segment entirely inside its zero k-range, as concatenated indices
  const int zt0 = p.nseg > 1 ? kt0 + (a.zk0 + 15) / 16 : 0;
  const int zt1 = p.nseg > 1 ? kt0 + a.zk1 / 16 : 0;
  const int zr_blocks = a.zero_rows / 8;  // member-local blocks entirely below zero_rows
  // warp w's part, first block (member-local) and block count
  auto wplace = [&](int w, int& part, int& fb, int& cnt) {
    part = w < pl.w0 ? 0 : 1;
    const int q = part ? w - pl.w0 : w;
    fb = pl.sb[part] + q * RB_FM;
    const int left = pl.nb[part] - q * RB_FM;
    cnt = left < RB_FM ? left : RB_FM;
  };
  auto skips = [&](int fb, int cnt, int g) {  // warp's blocks all exact zero on k-tile g
    return g >= zt0 && g < zt1 && fb + cnt <= zr_blocks;
  };

  if (tid == 0) {
    for (int s = 0; s < RB_STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, pl.nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  if (pl.nw == 0) return;

  if (warp == RB_WARPS) {  // producer
    if (lane == 0) {
      // per consumer warp: global first row, block count, compact smem slot, all-zero flag
      int wrow[RB_WARPS], wcnt[RB_WARPS], wslot[RB_WARPS];
      bool wz[RB_WARPS];
      int bytes_all = 0, bytes_nz = 0;
#pragma unroll
      for (int w = 0; w < RB_WARPS; ++w) {
        int part = 0, fb = 0, cnt = 0;
        if (w < pl.nw) wplace(w, part, fb, cnt);
        wrow[w] = pl.e[part] * p.M + fb * 8;
        wcnt[w] = cnt;
        wslot[w] = (part ? pl.nb[0] : 0) + (fb - pl.sb[part]);
        wz[w] = fb + cnt <= zr_blocks;
        bytes_all += cnt * 1024;
        if (!wz[w]) bytes_nz += cnt * 1024;
      }
      const int nparts = pl.nb[1] ? 2 : 1;
      for (int gk = 0; gk < ktot; ++gk) {
        const int st = gk % RB_STAGES;
        if (gk >= RB_STAGES) mbar_wait_cta(bar_empty + 8 * st, ((gk / RB_STAGES) - 1) & 1);
        const int s = gk < kt0 ? 0 : 1;
        const int kk = (s ? gk - kt0 : gk) * 16;
        const bool zt = gk >= zt0 && gk < zt1;
        const unsigned full = bar_full + 8 * st;
        mbar_expect_tx(full, (zt ? bytes_nz : bytes_all) + nparts * RB_B_BYTES);
        const unsigned dA = sbase + st * RB_STAGE;
#pragma unroll
        for (int w = 0; w < RB_WARPS; ++w) {
          if (wcnt[w] == 0 || (zt && wz[w])) continue;
          if (wcnt[w] == RB_FM) {
            tma_load_4d(dA + wslot[w] * 1024, &a.ta4[s], kk, wrow[w], 0, 0, full);
          } else {
            for (int x = 0; x < wcnt[w]; ++x)
              tma_load_4d(dA + (wslot[w] + x) * 1024, &a.ta[s], kk, wrow[w] + 8 * x, 0, 0, full);
          }
        }
        for (int part = 0; part < nparts; ++part)
          tma_load_4d(dA + RB_A_BYTES + part * RB_B_BYTES, &a.tb[s], kk, pl.e[part] * p.N, 0, 0,
                      full);
      }
    }
    return;
  }
  if (warp >= pl.nw) return;  // no blocks for this warp

  int part, fb, cnt;
  wplace(warp, part, fb, cnt);
  const int slot0 = (part ? pl.nb[0] : 0) + (fb - pl.sb[part]);
  const int g = lane >> 2, t4 = lane & 3;
  const unsigned ko0 = swz(g, 4 * t4), ko1 = swz(g, 4 * t4 + 2);
  double acc[RB_FM][RB_FN][2];
#pragma unroll
  for (int x = 0; x < RB_FM; ++x)
#pragma unroll
    for (int y = 0; y < RB_FN; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  auto kloop = [&](auto FMC) {  // FMC: this warp's block count, compile-time
    constexpr int F = decltype(FMC)::value;
    for (int gk = 0; gk < ktot; ++gk) {
      const int st = gk % RB_STAGES;
      mbar_wait_cta(bar_full + 8 * st, (gk / RB_STAGES) & 1);
      if (skips(fb, cnt, gk)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty + 8 * st);
        continue;
      }
      const unsigned char* sa = sgen + st * RB_STAGE + slot0 * 1024;
      const unsigned char* sbp = sgen + st * RB_STAGE + RB_A_BYTES + part * RB_B_BYTES;
      double af[F][4], bf[RB_FN][4];
#pragma unroll
      for (int x = 0; x < F; ++x) {
        const double2 u = *reinterpret_cast<const double2*>(sa + x * 1024 + ko0);
        const double2 v = *reinterpret_cast<const double2*>(sa + x * 1024 + ko1);
        af[x][0] = u.x; af[x][1] = u.y; af[x][2] = v.x; af[x][3] = v.y;
      }
#pragma unroll
      for (int y = 0; y < RB_FN; ++y) {
        const double2 u = *reinterpret_cast<const double2*>(sbp + y * 8 * 128 + ko0);
        const double2 v = *reinterpret_cast<const double2*>(sbp + y * 8 * 128 + ko1);
        bf[y][0] = u.x; bf[y][1] = u.y; bf[y][2] = v.x; bf[y][3] = v.y;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + 8 * st);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int x = 0; x < F; ++x)
#pragma unroll
          for (int y = 0; y < RB_FN; ++y)
            dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x][q], bf[y][q]);
    }
  };
  switch (cnt) {
    case 4: kloop(std::integral_constant<int, 4>{}); break;
    case 3: kloop(std::integral_constant<int, 3>{}); break;
    case 2: kloop(std::integral_constant<int, 2>{}); break;
    default: kloop(std::integral_constant<int, 1>{}); break;
  }
  // rows fb*8 .. (fb+cnt)*8 of member pl.e[part]; blocks past cnt hold zeros, not stored
#pragma unroll
  for (int x = 0; x < RB_FM; ++x)
    if (x < cnt)
      gemm_epilogue<1, RB_FN>(p, pl.e[part], 0, (fb + x) * 8 + g, 2 * t4,
                              reinterpret_cast<const double(&)[1][RB_FN][2]>(acc[x]));
}

// Eligibility: batch over nb1 >= 2 only, M % 8 == 0, N <= 32, 1-2 k-contiguous segments
// whose A rows share one stride and batch stride M * stride (a dense member-major stack,
// as T), B columns k-contiguous with batch stride N * column stride, TMA alignment, and at
// most RB_MAXB (< M / 8) blocks per SM so that a range spans at most two members.
static int num_sms() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    PE_CUDA_CHECK(cudaGetDevice(&dev));
    PE_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  return nsm;
}

// work weights of the two block kinds (k-tiles multiplied): wu below zero_rows, ww above
static void rb_weights(const GemmParams& p, int zero_rows, int zero_k0, int zero_k1, int& wu,
                       int& ww, int& zrb) {
  const int kt0 = (p.seg[0].K + 15) / 16, kt1 = p.nseg > 1 ? (p.seg[1].K + 15) / 16 : 0;
  const int nz = p.nseg > 1 ? std::max(0, zero_k1 / 16 - (zero_k0 + 15) / 16) : 0;
  ww = kt0 + kt1;
  wu = std::max(1, ww - nz);
  zrb = p.nseg > 1 ? std::min(std::max(zero_rows, 0) / 8, p.M / 8) : 0;
}

bool gemm_rowbalanced_eligible(const GemmParams& p, int zero_rows, int zero_k0, int zero_k1) {
  static const bool off = getenv("PE_GEMM_NO_ROWBAL") != nullptr;
  if (off || p.nb2 != 1 || p.nb1 < 2 || p.M % 8 || p.N > 8 * RB_FN || p.N < 1 || p.nseg < 1 ||
      p.nseg > 2 || p.nrm || p.Cin || !tma_ok(p))
    return false;
  for (int s = 0; s < p.nseg; ++s) {
    const Operand& A = p.seg[s].A;
    const Operand& B = p.seg[s].B;
    if (A.b1 != (long long)p.M * A.s0 || B.b1 != (long long)p.N * B.s1) return false;
  }
  const long long blocks = (long long)p.nb1 * (p.M / 8);
  if (blocks > INT32_MAX) return false;
  int wu, ww, zrb;
  rb_weights(p, zero_rows, zero_k0, zero_k1, wu, ww, zrb);
  const int mb = p.M / 8;
  const long long W = (long long)p.nb1 * ((long long)zrb * wu + (long long)(mb - zrb) * ww);
  const int grid = (int)std::min<long long>(num_sms(), blocks);
  // longest possible range: all of it in the cheaper kind, +2 for the rounding at both ends
  const double per = (double)W / grid / std::min(wu, ww) + 2.0;
  return per <= RB_MAXB && per <= mb;
}

void gemm_f64_rowbalanced(const GemmParams& p, int zero_rows, int zero_k0, int zero_k1,
                          cudaStream_t st) {
  if (!gemm_rowbalanced_eligible(p, zero_rows, zero_k0, zero_k1))
    throw Error{PE_ERR_ARG, "rowbalanced: shape not eligible"};
  const long long blocks = (long long)p.nb1 * (p.M / 8);
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(gemm_rowbal_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RB_SMEM));
    attr = true;
  }
  RowBalArgs a;
  memset(static_cast<void*>(&a), 0, sizeof(a));
  a.p = p;
  a.p.ksplit = 1;
  for (int s = 0; s < p.nseg; ++s) {
    const GemmSeg& g = p.seg[s];
    int use[2];
    // rows of all members as one 2-D extent (member-major stack)
    encode_operand(&a.ta[s], use, g.A.p, g.K, p.M * p.nb1, g.A.s0, 0, 1, 0, 1, 8);
    encode_operand(&a.ta4[s], use, g.A.p, g.K, p.M * p.nb1, g.A.s0, 0, 1, 0, 1, 8 * RB_FM);
    encode_operand(&a.tb[s], use, g.B.p, g.K, p.N * p.nb1, g.B.s1, 0, 1, 0, 1, 8 * RB_FN);
  }
  a.blocks = (int)blocks;
  a.zero_rows = zero_rows;
  a.zk0 = zero_k0;
  a.zk1 = zero_k1;
  rb_weights(p, zero_rows, zero_k0, zero_k1, a.wu, a.ww, a.zrb);
  const int grid = (int)std::min<long long>(num_sms(), blocks);
  launch_k(gemm_rowbal_kernel, dim3(grid), dim3((RB_WARPS + 1) * 32), RB_SMEM, st, a);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
}

// ----------------------------------------------------------------------------------------
// The same row-balanced step, J times in ONE cooperative launch (the ensemble fine chain):
//     X_{s+1} = T [X_s ; D_s] + c,   D_{s+1} = X_{s+1} - X_s
// Every CTA keeps its row range for all steps.  A range's B operand is the full state of its
// (at most two) members, written by the two or three CTAs that cover the member: after its
// epilogue a CTA's last consumer warp release-increments a per-member counter, and the
// producer lane admits step s+1's B tiles once the counters of its members show s+1 complete
// covers (then a proxy fence: the TMA engine reads what other SMs stored).  The producer
// streams step s+1's T tiles while the consumers are still in step s's epilogue, so T keeps
// coming from HBM across the step boundary; a launch per step left every SM idle for ~15 %
// of the step (CTA launch, pipeline fill, tail).  Ring phases run on across steps.
struct alignas(64) RowBalChainArgs {
  CUtensorMap ta[2][RB_FM];   // T segments, boxes of 8, 16, 24, 32 rows (a warp's blocks: one TMA)
  CUtensorMap tbx[3];         // X_in, bufX[0], bufX[1]
  CUtensorMap tbd[3];         // D_in (when present), bufD[0], bufD[1]
  GemmParams p;               // epilogue template: M, N, strides, bias
  int blocks;
  int zero_rows, zk0, zk1;
  int wu, ww, zrb;
  int J, has_d0;
  int wmode, share3;          // block-to-warp split: by work (1) or by count; SMSP 3 share / 2
  const double* X_in;
  double* X_out;
  double* bufX[2];
  double* bufD[2];
  unsigned* cnt;              // per member: covers that finished a step (zeroed before launch)
  const int* active;          // per member, or null: members with 0 are left out of the split
};
constexpr int RB_MAXE = 64;   // members per launch when an active mask is given

constexpr unsigned RB_SPIN_LIMIT = 1u << 26;

__global__ void __launch_bounds__((RB_WARPS + 1) * 32, 1)
    gemm_rowbal_chain_kernel(const __grid_constant__ RowBalChainArgs a) {
  extern __shared__ unsigned char smraw[];
  const unsigned sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const unsigned char* sgen = smraw + (sbase - smem_u32(smraw));
  const unsigned bar_full = sbase + RB_STAGES * RB_STAGE;
  const unsigned bar_empty = bar_full + RB_STAGES * 8;
  __shared__ unsigned done_tickets;
  __shared__ int ncov_s[2];
  // warp -> (part, first member-local block, block count).  The blocks of a part are spread
  // by work over its share of the 11 consumer warps (2-4 blocks each at cfg4) instead of
  // four per warp with the remainder on the last one: with 37 blocks, four per warp put 12
  // blocks on SMSP 0 and 8 on SMSPs 2 and 3 (the DMMA pipes are per SMSP)
  __shared__ short w_part[RB_WARPS], w_fb[RB_WARPS], w_cnt[RB_WARPS];
  __shared__ int nw_active;
  const GemmParams& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Frozen (converged) members take no part: the rows of the ACTIVE members, in member order,
  // are what the CTAs split, so a sweep costs in proportion to the members still iterating.
  __shared__ short act_s[RB_MAXE];
  __shared__ int nact_s;
  if (tid == 0) {
    int n = 0;
    if (a.active) {
      for (int e = 0; e < p.nb1; ++e)
        if (a.active[e]) act_s[n++] = (short)e;
    } else {
      n = p.nb1;
    }
    nact_s = n;
  }
  __syncthreads();
  RbGeom geo = rb_geom(a);
  geo.blocks = nact_s * (p.M / 8);
  const RbPlan pl = rb_plan(geo);
  // plan member index -> member (identity without a mask)
  auto member = [&](int e) { return a.active ? (int)act_s[e < nact_s ? e : 0] : e; };
  const int em[2] = {member(pl.e[0]), member(pl.e[1])};
  const int kt0 = (p.seg[0].K + 15) / 16, kt1 = (p.seg[1].K + 15) / 16;
  const int zt0 = kt0 + (a.zk0 + 15) / 16, zt1 = kt0 + a.zk1 / 16;
  const int zr_blocks = a.zero_rows / 8;
  const int mb = p.M / 8;
  auto wplace = [&](int w, int& part, int& fb, int& cnt) {
    part = w_part[w];
    fb = w_fb[w];
    cnt = w_cnt[w];
  };
  auto skips = [&](int fb, int cnt, int g) {
    return g >= zt0 && g < zt1 && fb + cnt <= zr_blocks;
  };
  const int nparts = pl.nb[1] ? 2 : 1;

  if (tid == 0) {
    // Work-weighted: a block below the zero-row boundary multiplies wu k-tiles, any other ww;
    // a warp on the producer's SMSP (two consumer warps instead of three) takes a 3/2 share.
    auto bw = [&](int part, int b) {
      return a.wmode ? (pl.sb[part] + b < a.zrb ? a.wu : a.ww) : 1;
    };
    long long Wp[2] = {0, 0};
    for (int part = 0; part < 2; ++part)
      for (int b = 0; b < pl.nb[part]; ++b) Wp[part] += bw(part, b);
    const int nb0 = pl.nb[0], nb1 = pl.nb[1];
    int wp[2] = {0, 0};
    if (nb0 + nb1 > 0) {
      if (nb1 == 0) {
        wp[0] = min(RB_WARPS, nb0);
      } else {
        int w0 = (int)((RB_WARPS * Wp[0] + (Wp[0] + Wp[1]) / 2) / (Wp[0] + Wp[1]));
        w0 = max(w0, (nb0 + RB_FM - 1) / RB_FM);
        w0 = min(w0, RB_WARPS - (nb1 + RB_FM - 1) / RB_FM);
        w0 = max(1, min(w0, nb0));
        wp[0] = w0;
        wp[1] = min(RB_WARPS - w0, nb1);
      }
    }
    int w = 0, active = 0;
    for (int part = 0; part < 2; ++part) {
      const int nbp = pl.nb[part], n = wp[part];
      if (n == 0) continue;
      int S = 0;
      for (int i = 0; i < n; ++i) S += ((w + i) & 3) == (RB_WARPS & 3) ? a.share3 : 2;
      int pos = 0, cs = 0;
      long long cum = 0;
      for (int i = 0; i < n; ++i) {
        cs += ((w + i) & 3) == (RB_WARPS & 3) ? a.share3 : 2;
        const long long target = Wp[part] * cs / S;
        const int lo = max(0, (nbp - pos) - RB_FM * (n - 1 - i)), hi = min(RB_FM, nbp - pos);
        int c = 0;
        long long ws = 0;
        while (c < hi) {
          const int wb = bw(part, pos + c);
          if (c >= lo && 2 * (cum + ws) + wb > 2 * target) break;
          ws += wb;
          ++c;
        }
        w_part[w + i] = (short)part;
        w_fb[w + i] = (short)(pl.sb[part] + pos);
        w_cnt[w + i] = (short)c;
        active += c > 0;
        pos += c;
        cum += ws;
      }
      w += n;
    }
    nw_active = active;
    for (; w < RB_WARPS; ++w) {
      w_part[w] = 0;
      w_fb[w] = (short)pl.sb[0];
      w_cnt[w] = 0;
    }
    for (int s = 0; s < RB_STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, nw_active);
    }
    done_tickets = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    // covers of this range's members: CTAs whose (non-empty) range meets the member's blocks
    for (int part = 0; part < 2; ++part) {
      const long long m0 = (long long)pl.e[part] * mb, m1 = m0 + mb;
      int n = 0;
      for (int c0 = 0; c0 < (int)gridDim.x; c0 += 32) {  // small ensembles: many covers
        const int c = c0 + lane;
        bool hit = false;
        if (c < (int)gridDim.x) {
          long long b0, b1;
          rb_range(geo, c, b0, b1);
          hit = b1 > b0 && b0 < m1 && b1 > m0;
        }
        n += __popc(__ballot_sync(0xffffffffu, hit));
      }
      if (lane == 0) ncov_s[part] = n;
    }
  }
  __syncthreads();
  const int nwa = nw_active;
  if (nwa == 0) return;
  const int J = a.J;

  if (warp == RB_WARPS) {  // producer
    if (lane == 0) {
      int wrow[RB_WARPS], wcnt[RB_WARPS], wslot[RB_WARPS];
      bool wz[RB_WARPS];
      int bytes_all = 0, bytes_nz = 0;
#pragma unroll
      for (int w = 0; w < RB_WARPS; ++w) {
        int part = 0, fb = 0, cnt = 0;
        wplace(w, part, fb, cnt);
        wrow[w] = em[part] * p.M + fb * 8;
        wcnt[w] = cnt;
        wslot[w] = (part ? pl.nb[0] : 0) + (fb - pl.sb[part]);
        wz[w] = fb + cnt <= zr_blocks;
        bytes_all += cnt * 1024;
        if (!wz[w]) bytes_nz += cnt * 1024;
      }
      const unsigned need0 = (unsigned)ncov_s[0], need1 = (unsigned)ncov_s[1];
      int gidx = 0;  // k-tiles issued so far, over all steps
      for (int s = 0; s < J; ++s) {
        const bool two = s > 0 || a.has_d0;
        const int ktot = two ? kt0 + kt1 : kt0;
        const int bsel = s == 0 ? 0 : 1 + ((s - 1) & 1);
        bool admitted = s == 0;
        for (int gk = 0; gk < ktot; ++gk, ++gidx) {
          const int st = gidx % RB_STAGES;
          if (gidx >= RB_STAGES) mbar_wait_cta(bar_empty + 8 * st, ((gidx / RB_STAGES) - 1) & 1);
          const int sg = gk < kt0 ? 0 : 1;
          const int kk = (sg ? gk - kt0 : gk) * 16;
          const bool zt = gk >= zt0 && gk < zt1;
          const unsigned full = bar_full + 8 * st;
          mbar_expect_tx(full, (zt ? bytes_nz : bytes_all) + nparts * RB_B_BYTES);
          const unsigned dA = sbase + st * RB_STAGE;
#pragma unroll
          for (int w = 0; w < RB_WARPS; ++w) {
            if (wcnt[w] == 0 || (zt && wz[w])) continue;
            tma_load_4d(dA + wslot[w] * 1024, &a.ta[sg][wcnt[w] - 1], kk, wrow[w], 0, 0, full);
          }
          if (!admitted) {
            // every cover of both members has stored step s - 1 (T tiles above did not wait)
            unsigned spins = 0;
            for (;;) {
              unsigned c0v, c1v = 0xffffffffu;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c0v) : "l"(a.cnt + em[0]) : "memory");
              if (nparts > 1)
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c1v) : "l"(a.cnt + em[1]) : "memory");
              if (c0v >= (unsigned)s * need0 && (nparts < 2 || c1v >= (unsigned)s * need1)) break;
              if (++spins > RB_SPIN_LIMIT) __trap();
            }
            asm volatile("fence.proxy.async;" ::: "memory");  // generic-proxy stores -> TMA reads
            admitted = true;
          }
          const CUtensorMap* tb = sg ? &a.tbd[bsel] : &a.tbx[bsel];
          for (int part = 0; part < nparts; ++part)
            tma_load_4d(dA + RB_A_BYTES + part * RB_B_BYTES, tb, kk, em[part] * p.N, 0, 0, full);
        }
      }
    }
    return;
  }
  int part, fb, cnt;
  wplace(warp, part, fb, cnt);
  if (cnt == 0) return;  // no blocks for this warp
  const int slot0 = (part ? pl.nb[0] : 0) + (fb - pl.sb[part]);
  const int g = lane >> 2, t4 = lane & 3;
  const unsigned ko0 = swz(g, 4 * t4), ko1 = swz(g, 4 * t4 + 2);
  int gbase = 0;
  for (int s = 0; s < J; ++s) {
    const bool two = s > 0 || a.has_d0;
    const int ktot = two ? kt0 + kt1 : kt0;
    const bool last = s == J - 1;
    double acc[RB_FM][RB_FN][2];
#pragma unroll
    for (int x = 0; x < RB_FM; ++x)
#pragma unroll
      for (int y = 0; y < RB_FN; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    auto kloop = [&](auto FMC) {  // FMC: this warp's block count, compile-time
      constexpr int F = decltype(FMC)::value;
      for (int gk = 0; gk < ktot; ++gk) {
        const int gidx = gbase + gk;
        const int st = gidx % RB_STAGES;
        mbar_wait_cta(bar_full + 8 * st, (gidx / RB_STAGES) & 1);
        if (skips(fb, cnt, gk)) {
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_empty + 8 * st);
          continue;
        }
        const unsigned char* sa = sgen + st * RB_STAGE + slot0 * 1024;
        const unsigned char* sbp = sgen + st * RB_STAGE + RB_A_BYTES + part * RB_B_BYTES;
        double af[F][4], bf[RB_FN][4];
#pragma unroll
        for (int x = 0; x < F; ++x) {
          const double2 u = *reinterpret_cast<const double2*>(sa + x * 1024 + ko0);
          const double2 v = *reinterpret_cast<const double2*>(sa + x * 1024 + ko1);
          af[x][0] = u.x; af[x][1] = u.y; af[x][2] = v.x; af[x][3] = v.y;
        }
#pragma unroll
        for (int y = 0; y < RB_FN; ++y) {
          const double2 u = *reinterpret_cast<const double2*>(sbp + y * 8 * 128 + ko0);
          const double2 v = *reinterpret_cast<const double2*>(sbp + y * 8 * 128 + ko1);
          bf[y][0] = u.x; bf[y][1] = u.y; bf[y][2] = v.x; bf[y][3] = v.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty + 8 * st);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
          for (int x = 0; x < F; ++x)
#pragma unroll
            for (int y = 0; y < RB_FN; ++y)
              dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x][qq], bf[y][qq]);
      }
    };
    switch (cnt) {
      case 4: kloop(std::integral_constant<int, 4>{}); break;
      case 3: kloop(std::integral_constant<int, 3>{}); break;
      case 2: kloop(std::integral_constant<int, 2>{}); break;
      default: kloop(std::integral_constant<int, 1>{}); break;
    }
    gbase += ktot;
    // epilogue (gemm_epilogue's arithmetic for alpha = 1, no Cin): C = acc + bias,
    // D = C - X_s; only the three pointers change from step to step
    {
      const long long cb = (long long)em[part] * p.c_b1;
      double* C = (last ? a.X_out : a.bufX[s & 1]) + cb;
      double* D = last ? nullptr : a.bufD[s & 1] + cb;
      const double* Xp = last ? nullptr : (s == 0 ? a.X_in : a.bufX[(s - 1) & 1]) + cb;
      const double* bias = p.bias ? p.bias + (long long)em[part] * p.bias_b1 : nullptr;
#pragma unroll
      for (int x = 0; x < RB_FM; ++x) {
        if (x >= cnt) continue;
        const int gi = (fb + x) * 8 + g;
        const long long ro = gi * p.c_i;
        double pre[RB_FN][2];
#pragma unroll
        for (int b = 0; b < RB_FN; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gj = 2 * t4 + b * 8 + h;
            pre[b][h] = (Xp && gj < p.N) ? Xp[ro + gj * p.c_j] : 0.0;
          }
        const double bv = bias ? bias[gi] : 0.0;
#pragma unroll
        for (int b = 0; b < RB_FN; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gj = 2 * t4 + b * 8 + h;
            if (gj >= p.N) continue;
            const long long off = ro + gj * p.c_j;
            double v = acc[x][b][h];
            if (bias) v = __dadd_rn(v, bv);
            C[off] = v;
            if (D) D[off] = __dsub_rn(v, pre[b][h]);
          }
      }
    }
    if (!last) {
      // the last consumer warp to finish publishes the step for both members (its release at
      // gpu scope is cumulative over the other warps' cta-scope releases)
      __syncwarp();
      if (lane == 0) {
        unsigned t;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(t) : "r"(smem_u32(&done_tickets)) : "memory");
        if (t + 1 == (unsigned)nwa * (unsigned)(s + 1)) {
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.cnt + em[0]) : "memory");
          if (nparts > 1)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.cnt + em[1]) : "memory");
        }
      }
    }
  }
}

bool gemm_rowbalanced_chain_eligible(const GemmParams& p2, int zero_rows, int zero_k0, int zero_k1) {
  static const bool off = getenv("PE_ROWBAL_NO_CHAIN") != nullptr;
  if (off || p2.nseg != 2 || p2.alpha != 1.0 || p2.Cin) return false;
  // the range split of the two-segment step is used for every step (also a one-segment
  // first step), and the whole grid must be co-resident
  const long long blocks = (long long)p2.nb1 * (p2.M / 8);
  return gemm_rowbalanced_eligible(p2, zero_rows, zero_k0, zero_k1) && blocks >= num_sms();
}

void gemm_f64_rowbalanced_chain(const GemmParams& p2, int zero_rows, int zero_k0, int zero_k1, int J,
                                const double* X_in, const double* D_in, double* const bufX[2],
                                double* const bufD[2], double* X_out, unsigned* cnt,
                                const int* active, cudaStream_t st) {
  if (!gemm_rowbalanced_chain_eligible(p2, zero_rows, zero_k0, zero_k1))
    throw Error{PE_ERR_ARG, "rowbalanced chain: shape not eligible"};
  const long long blocks = (long long)p2.nb1 * (p2.M / 8);
  static bool attr = false;
  if (!attr) {
    PE_CUDA_CHECK(cudaFuncSetAttribute(gemm_rowbal_chain_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RB_SMEM));
    attr = true;
  }
  RowBalChainArgs a;
  memset(static_cast<void*>(&a), 0, sizeof(a));
  a.p = p2;
  a.p.ksplit = 1;
  int use[2];
  for (int s = 0; s < 2; ++s) {
    const GemmSeg& g = p2.seg[s];
    for (int f = 1; f <= RB_FM; ++f)
      encode_operand(&a.ta[s][f - 1], use, g.A.p, g.K, p2.M * p2.nb1, g.A.s0, 0, 1, 0, 1, 8 * f);
  }
  const long long bs1 = p2.seg[0].B.s1;
  const double* bx[3] = {X_in, bufX[0], bufX[1]};
  const double* bd[3] = {D_in ? D_in : bufD[0], bufD[0], bufD[1]};
  for (int i = 0; i < 3; ++i) {
    encode_operand(&a.tbx[i], use, bx[i], p2.seg[0].K, p2.N * p2.nb1, bs1, 0, 1, 0, 1, 8 * RB_FN);
    encode_operand(&a.tbd[i], use, bd[i], p2.seg[1].K, p2.N * p2.nb1, bs1, 0, 1, 0, 1, 8 * RB_FN);
  }
  a.blocks = (int)blocks;
  a.zero_rows = zero_rows;
  a.zk0 = zero_k0;
  a.zk1 = zero_k1;
  rb_weights(p2, zero_rows, zero_k0, zero_k1, a.wu, a.ww, a.zrb);
  a.J = J;
  a.has_d0 = D_in != nullptr;
  // measured at cfg4 (GEMM ms per iteration): by count, producer-SMSP share 3/2: 3.30; share
  // 1: 3.62; by work, share 3/2: 3.32; share 1: 3.50; share 2: 3.38
  static const int wmode = getenv("PE_RB_WMODE") ? atoi(getenv("PE_RB_WMODE")) : 0;
  static const int share3 = getenv("PE_RB_SHARE3") ? atoi(getenv("PE_RB_SHARE3")) : 3;
  a.wmode = wmode;
  a.share3 = share3;
  a.X_in = X_in;
  a.X_out = X_out;
  a.bufX[0] = bufX[0];
  a.bufX[1] = bufX[1];
  a.bufD[0] = bufD[0];
  a.bufD[1] = bufD[1];
  a.cnt = cnt;
  a.active = p2.nb1 <= RB_MAXE ? active : nullptr;
  PE_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * p2.nb1, st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3((RB_WARPS + 1) * 32);
  cfg.dynamicSmemBytes = RB_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other: all co-resident
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_rowbal_chain_kernel, a));
  ++g_launches;
}

void gemm_f64(const GemmParams& p, cudaStream_t st) {
  if (p.M <= 0 || p.N <= 0 || p.nb1 * p.nb2 <= 0) return;
  bool ak = true, bk = true;
  for (int s = 0; s < p.nseg; ++s) {
    const bool sa = (p.seg[s].A.s1 == 1), sb = (p.seg[s].B.s0 == 1);
    if (s == 0) {
      ak = sa;
      bk = sb;
    } else if (sa != ak || sb != bk) {
      throw Error{PE_ERR_ARG, "gemm_f64: segments with mixed operand layouts"};
    }
  }
  const long long batch = (long long)p.nb1 * p.nb2;
  const long long tiles64 = (long long)((p.M + 63) / 64) * ((p.N + 63) / 64) * batch;
  const long long tiles_n32 = (long long)((p.M + 127) / 128) * ((p.N + 31) / 32) * batch;
  static const bool no_fast = getenv("PE_GEMM_GENERIC") != nullptr;
  const int lay = no_fast ? -1 : fast_layout(p);
  // skinny launch (few row tiles x batch): split K over extra CTAs, decided from
  // (M, K, batch) only so that any column count gives the same arithmetic
  if (lay >= 0 && p.ws && !p.nrm) {
    const long long mt = (long long)((p.M + 63) / 64) * batch;
    int ktiles = 0;
    for (int sgi = 0; sgi < p.nseg; ++sgi) ktiles += (p.seg[sgi].K + 31) / 32;
    int ks = (int)std::min<long long>(8, 148 / std::max<long long>(1, mt));
    ks = std::min(ks, ktiles / 2);  // >= 2 k-tiles of 32 per split
    if (ks >= 2 && (size_t)ks * batch * p.M * p.N <= p.ws_doubles) {
      GemmParams q = p;
      q.ksplit = ks;
      if (lay == 0)
        launch_fast<2, 2, 4, 4, 32, 3, false>(q, st);
      else
        launch_fast<2, 2, 4, 4, 32, 3, true>(q, st);
      const long long total = (long long)batch * p.M * p.N;
      launch_k(splitk_reduce_kernel, dim3((unsigned)std::min<long long>(148 * 8, (total + 255) / 256)),
               dim3(256), 0, st, q);
      ++g_launches;
      PE_CUDA_CHECK(cudaGetLastError());
      return;
    }
  }
  // TMA pipeline: measured faster than the cp.async kernels only for many skinny batched
  // products (the shifted solves: N <= 128 per batch, long K); slower on the wide rhs / g /
  // norm / ensemble-step shapes (tools/gemm_bench.py, profiles/r01/README.md)
  static const bool tma_all = getenv("PE_GEMM_TMA_ALL") != nullptr;  // tuning only
  static const bool no_big_tma = getenv("PE_GEMM_NO_BIG_TMA") != nullptr;
  const bool tma_shape = (batch >= 16 && p.N <= 128 && p.seg[0].K >= 512) || tma_all;
  // Many-wave products with a long K (the config-3 rhs / h / norm products: 12800 tiles of
  // 64 x 64, K = 8192): the TMA producer pipeline with 64 x 64 tiles measured 35.7 TF/s
  // against 34.5 for the cp.async kernel (cuBLAS 36.0, tools/gemm_bench.py); the wide
  // medium-size modal shapes of config 2 (285 tiles, one wave) stay on cp.async.
  int ktiles16 = 0;
  for (int sgi = 0; sgi < p.nseg; ++sgi) ktiles16 += (p.seg[sgi].K + 15) / 16;
  const bool big = !no_big_tma && p.M >= 256 && p.N >= 256 && tiles64 >= 8 * 148 && ktiles16 >= 128;
  if (lay == 0 && big && tma_ok(p)) {
    launch_tma<2, 2, 4, 4, 4>(p, st);
  } else if (lay == 0 && (tiles64 >= 96 || tiles_n32 >= 96) && tma_shape && tma_ok(p)) {
    launch_tma_best(p, st);
  } else if (lay >= 0 && (tiles64 >= 96 || tiles_n32 >= 96)) {
    // pick the tile / pipeline variant with the best wave-quantised cost; the choice is a
    // function of the shape only and never changes the arithmetic
    static const int forced = getenv("PE_GEMM_VARIANT") ? atoi(getenv("PE_GEMM_VARIANT")) : -1;
    int best = (lay == 0) ? choose_variant<false>(p) : choose_variant<true>(p);
    if (forced >= 0 && forced < kMaxVariant && forced != 4) best = forced;  // tuning only
    static const bool trace = getenv("PE_GEMM_TRACE") != nullptr;
    if (trace)
      fprintf(stderr, "pe_gemm M=%d N=%d K=%d batch=%lld lay=%d variant=%d\n", p.M, p.N,
              p.seg[0].K, batch, lay, best);
    int ktiles = 0;
    for (int sgi = 0; sgi < p.nseg; ++sgi) ktiles += (p.seg[sgi].K + 15) / 16;
    const bool pre = ktiles >= 256;  // long K: precomputed load descriptors
    if (lay == 0)
      launch_variant<false>(best, p, st, pre);
    else
      launch_variant<true>(best, p, st);
  } else if (tiles64 >= 2 * 148) {
    launch_cfg<64, 64, 16, 32, 32>(p, ak, bk, st);
  } else {
    launch_cfg<32, 32, 16, 16, 16>(p, ak, bk, st);
  }
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe
