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
#include <stdexcept>

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
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// AK: A is k-contiguous (s1 == 1); BKC: B is k-contiguous (s0 == 1).
template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKC>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    gemm_f64_kernel(const __grid_constant__ GemmParams p) {
  constexpr int WARPS_M = BM / WM;
  constexpr int NT = WARPS_M * (BN / WN) * 32;
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int SK = BK + 4;  // row stride in doubles: 16-lane half-warps hit distinct banks
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

  if (ntile > 0) {
    load_tile(0, 0);
    cp_async_commit();
    for (int t = 0; t < ntile; ++t) {
      const int buf = t & 1;
      if (t + 1 < ntile) {
        load_tile(t + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* as = &As[buf][(wm * WM + g) * SK + t4];
      const double* bs = &Bs[buf][(wn * WN + g) * SK + t4];
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[FM], bf[FN];
#pragma unroll
        for (int a = 0; a < FM; ++a) af[a] = as[a * 8 * SK + kk];
#pragma unroll
        for (int b = 0; b < FN; ++b) bf[b] = bs[b * 8 * SK + kk];
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
          for (int b = 0; b < FN; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
      __syncthreads();
    }
  }

  // fused epilogue
  const long long cb = z1 * p.c_b1 + z2 * p.c_b2;
  double* C = p.C + cb;
  const double* Cin = p.Cin ? p.Cin + cb : nullptr;
  double* D = p.D ? p.D + cb : nullptr;
  const double* Xp = p.Xp ? p.Xp + cb : nullptr;
  const double* bias = p.bias ? p.bias + z1 * p.bias_b1 + z2 * p.bias_b2 : nullptr;
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int gi = i0 + wm * WM + a * 8 + g;
    if (gi >= p.M) continue;
    const double bv = bias ? bias[gi] : 0.0;
#pragma unroll
    for (int b = 0; b < FN; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = j0 + wn * WN + b * 8 + 2 * t4 + h;
        if (gj >= p.N) continue;
        const long long off = gi * p.c_i + gj * p.c_j;
        double v = (p.alpha == 1.0) ? acc[a][b][h] : __dmul_rn(p.alpha, acc[a][b][h]);
        if (Cin) v = __dadd_rn(v, (p.beta == 1.0) ? Cin[off] : __dmul_rn(p.beta, Cin[off]));
        if (bias) v = __dadd_rn(v, bv);
        C[off] = v;
        if (D) D[off] = __dsub_rn(v, Xp[off]);
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN>
static void launch_cfg(const GemmParams& p, bool ak, bool bk, cudaStream_t st) {
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.nb1 * p.nb2);
  dim3 block((BM / WM) * (BN / WN) * 32);
  if (ak && bk)
    gemm_f64_kernel<BM, BN, BK, WM, WN, true, true><<<grid, block, 0, st>>>(p);
  else if (ak && !bk)
    gemm_f64_kernel<BM, BN, BK, WM, WN, true, false><<<grid, block, 0, st>>>(p);
  else if (!ak && bk)
    gemm_f64_kernel<BM, BN, BK, WM, WN, false, true><<<grid, block, 0, st>>>(p);
  else
    gemm_f64_kernel<BM, BN, BK, WM, WN, false, false><<<grid, block, 0, st>>>(p);
  ++g_launches;
}

double gemm_flops(const GemmParams& p) {
  double k = 0;
  for (int s = 0; s < p.nseg; ++s) k += p.seg[s].K;
  return 2.0 * p.M * (double)p.N * k * p.nb1 * p.nb2;
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
  if (tiles64 >= 2 * 148)
    launch_cfg<64, 64, 16, 32, 32>(p, ak, bk, st);
  else
    launch_cfg<32, 32, 16, 16, 16>(p, ak, bk, st);
  PE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pe
