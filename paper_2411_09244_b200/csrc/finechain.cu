// Fine reference solve for large fine grids: block-tridiagonal chain solver.
//
// reference_solve (fem.py:292-318) applies (M/dt + A)^-1 once per backward-Euler step with a
// sparse LU.  K = M/dt + A of the Q1 grid is banded (half-bandwidth w = nodes per grid row
// + 1), so with blocks of bs >= w rows it is block tridiagonal, K = tridiag(L_i, D_i, U_i),
// and the block factorisation
//     S_0 = D_0,   S_i = D_i - L_i S_{i-1}^-1 U_{i-1},   P_i = S_i^-1  (dense bs x bs)
// turns a solve K x = v into two sweeps of nb dependent block steps:
//     forward   y_i = v_i - L_i z_{i-1},       z_i = P_i y_i
//     backward  x_i = z_i - P_i (U_i x_{i+1}), x_{nb-1} = z_{nb-1}
// L_i / U_i keep their sparse rows (<= a few entries per row); only P_i is dense.  Per step
// the solver streams 2 nb bs^2 doubles (268 MB at the config-3 grid, n = 65025, bs = 256)
// instead of the packed dense inverse's n^2 / 2 (16.9 GB): 63x fewer bytes, a 0.13 GB
// operator instead of 17 GB, ~0.1 s of setup instead of ~20 s, and no 65535-node cap.
//
// The sweeps are latency chains, so ONE thread-block cluster of 16 CTAs runs them: CTA c
// owns rows [c rpc, (c+1) rpc) of every block.  Per block step every CTA (1) forms the
// full sparse vector y_i (or U_i x_{i+1}) redundantly from the previous step's broadcast
// vector, (2) dots its own rows of P_i -- streamed by cp.async.bulk into a shared-memory
// ring that runs several block steps ahead -- with it, (3) writes its rpc results into
// every peer's receive buffer by st.async, completing on the receiver's mbarrier: the
// chain has no cluster barrier (the double-buffered receive is ordered by the data flow
// itself).  z_i stays in the owner's shared memory for the backward sweep.
//
// The block inverses come from libpe's own LU (batchlu.cu).  Deterministic: fixed-order
// dot products and shuffles.

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "finescale.h"
#include "mbar.cuh"
#include "pe.h"
#include "pe_internal.h"

namespace pe {

namespace cg = cooperative_groups;

namespace {

constexpr int CH_CS = 16;        // cluster size
constexpr int CH_T = 256;        // threads per CTA
constexpr int CH_W = CH_T / 32;  // warps
constexpr int CH_EW = 8;         // max off-diagonal-block entries per row
constexpr unsigned CH_CHUNK = 32 * 1024;

template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  explicit Buf(size_t count) : n(count) {
    if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error{PE_ERR_NOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed"};
    }
  }
  ~Buf() { cudaFree(p); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

struct ChainArgs {
  int n, bs, nb, rpc;      // rows, block size, blocks, rows per CTA
  int rc, npc, stages;     // rows per ring chunk, chunks per slice, ring depth
  const double* P;         // nb x bs x bs row-major block inverses
  const int* lidx;         // n_pad x CH_EW column-in-previous-block (or -1)
  const double* lval;
  const int* uidx;         // n_pad x CH_EW column-in-next-block (or -1)
  const double* uval;
  const double* v;         // n_pad right-hand side (zero past n)
  double* x;               // n solution
};

__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void st_async_b64(unsigned remote_addr, double x, unsigned remote_bar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   remote_addr),
               "l"(__double_as_longlong(x)), "r"(remote_bar)
               : "memory");
}

__global__ void __launch_bounds__(CH_T, 1) fine_chain_kernel(const __grid_constant__ ChainArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bs = a.bs, nb = a.nb, rpc = a.rpc, rc = a.rc, npc = a.npc, ST = a.stages;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                 // ST x rc x bs
  double* recv = ring + (size_t)ST * rc * bs;                         // 2 x bs
  double* full = recv + 2 * bs;                                       // bs (this step's vector)
  double* zloc = full + bs;                                           // nb x rpc
  __shared__ __align__(8) unsigned long long bar[8];
  __shared__ __align__(8) unsigned long long rbar[2];  // receive barriers, by step parity
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(smem_u32(&bar[s]), 1);
    mbar_init(smem_u32(&rbar[0]), 1);
    mbar_init(smem_u32(&rbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned chunk_bytes = (unsigned)(rc * bs * sizeof(double));
  const int steps = 2 * nb - 1;            // forward 0 .. nb-1, backward nb-2 .. 0
  const int G = steps * npc;               // ring chunks in consumption order
  auto block_of = [&](int step) { return step < nb ? step : 2 * nb - 2 - step; };
  auto issue = [&](int g) {
    const int step = g / npc, part = g - step * npc;
    const double* src = a.P + ((size_t)block_of(step) * bs + (size_t)rank * rpc + (size_t)part * rc) * bs;
    const unsigned b = smem_u32(&bar[g % ST]);
    mbar_expect_tx(b, chunk_bytes);
    bulk_load(smem_u32(ring + (size_t)(g % ST) * rc * bs), src, chunk_bytes, b);
  };
  if (tid == 0)
    for (int g = 0; g < ST && g < G; ++g) issue(g);
  // every CTA must have started before any peer writes into its receive buffers
  cl.sync();

  // sparse rows of the coming step, prefetched one step ahead (registers)
  int pidx[2][CH_EW];
  double pval[2][CH_EW], pv[2];
  auto prefetch = [&](int step) {
    const bool fwd = step < nb;
    const int blk = block_of(step);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = tid + h * CH_T;
      if (r < bs) {
        const size_t row = (size_t)blk * bs + r;
        const int* ip = (fwd ? a.lidx : a.uidx) + row * CH_EW;
        const double* vp = (fwd ? a.lval : a.uval) + row * CH_EW;
#pragma unroll
        for (int e = 0; e < CH_EW; ++e) {
          pidx[h][e] = ip[e];
          pval[h][e] = vp[e];
        }
        pv[h] = fwd ? a.v[row] : 0.0;
      }
    }
  };
  prefetch(0);
  int g = 0;
  for (int step = 0; step < steps; ++step) {
    const bool fwd = step < nb;
    const int blk = block_of(step);
    const double* prev = recv + (size_t)((step + 1) & 1) * bs;  // written during step - 1
    double* next = recv + (size_t)(step & 1) * bs;
    // this step's receive barrier: bs doubles from the 16 CTAs (own rows included)
    if (tid == 0) mbar_expect_tx(smem_u32(&rbar[step & 1]), (unsigned)(bs * sizeof(double)));
    // (1) full vector: y_i = v_i - L_i z_{i-1}  or  t_i = U_i x_{i+1}
    const bool has_prev = step > 0;
    if (has_prev) mbar_wait(smem_u32(&rbar[(step + 1) & 1]), ((step - 1) >> 1) & 1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = tid + h * CH_T;
      if (r < bs) {
        double acc = 0.0;
        if (has_prev) {
#pragma unroll
          for (int e = 0; e < CH_EW; ++e)
            if (pidx[h][e] >= 0) acc = fma(pval[h][e], prev[pidx[h][e]], acc);
        }
        full[r] = fwd ? pv[h] - acc : acc;
      }
    }
    if (step + 1 < steps) prefetch(step + 1);
    __syncthreads();  // full[] complete; every warp is past the previous step's ring chunk
    if (npc == 1 && tid == 0 && step > 0 && g - 1 + ST < G) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(g - 1 + ST);
    }
    // (2) own rows of P_i times the full vector, chunk by chunk; (3) broadcast.  No cluster
    // barrier: a peer's step s+2 stores into the buffer this CTA reads in step s+1 only
    // after it received this CTA's step s+1 rows, i.e. after that read.
    const unsigned next_u32 = smem_u32(next), rbar_u32 = smem_u32(&rbar[step & 1]);
    for (int part = 0; part < npc; ++part, ++g) {
      mbar_wait_cta(smem_u32(&bar[g % ST]), (g / ST) & 1);
      const double* tile = ring + (size_t)(g % ST) * rc * bs;
      // two rows per warp pass, one per half-warp (16 lanes x 16-byte loads: conflict free)
      const int half = lane >> 4, hl = lane & 15;
      for (int r2 = 2 * warp; r2 < rc; r2 += 2 * CH_W) {
        const int rr = r2 + half;
        const bool live = rr < rc;
        const double2* row = reinterpret_cast<const double2*>(tile + (size_t)(live ? rr : r2) * bs);
        const double2* f2 = reinterpret_cast<const double2*>(full);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int k = hl; k < bs / 2; k += 32) {  // bs % 64 == 0: both strides in range
          const double2 p = row[k], f = f2[k], q = row[k + 16], h2 = f2[k + 16];
          s0 = fma(p.x, f.x, s0);
          s1 = fma(p.y, f.y, s1);
          s2 = fma(q.x, h2.x, s2);
          s3 = fma(q.y, h2.y, s3);
        }
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const int lr = part * rc + (live ? rr : r2);  // local row
        double val;
        if (fwd) {
          val = s;  // z_i
          if (hl == 0 && live) zloc[(size_t)blk * rpc + lr] = val;
        } else {
          val = zloc[(size_t)blk * rpc + lr] - s;  // x_i
        }
        // each half-warp's 16 lanes store its row to the 16 CTAs
        if (live)
          st_async_b64(map_rank(next_u32 + (unsigned)((rank * rpc + lr) * sizeof(double)), hl), val,
                       map_rank(rbar_u32, hl));
        const int grow = blk * bs + rank * rpc + lr;
        if (hl == 0 && live && grow < a.n && (!fwd || blk == nb - 1)) a.x[grow] = val;
      }
      if (npc > 1) {
        __syncthreads();  // chunk fully read
        if (tid == 0 && g + ST < G) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(g + ST);
        }
      }
    }
  }
  // the last step's rows: nobody exits while a peer may still store into its buffers
  mbar_wait(smem_u32(&rbar[(steps - 1) & 1]), ((steps - 1) >> 1) & 1);
  cl.sync();
}

// dense diagonal blocks (row-major, identity on the padding rows) from the merged CSR of K
__global__ void chain_scatter_diag(int n, int bs, int nb, const int* kp, const int* ki,
                                   const double* kv, double* D) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb * bs) return;
  const int blk = r / bs;
  double* row = D + (size_t)r * bs;
  if (r >= n) {
    row[r - blk * bs] = 1.0;
    return;
  }
  for (int t = kp[r]; t < kp[r + 1]; ++t) {
    const int c = ki[t];
    if (c / bs == blk) row[c - blk * bs] = kv[t];
  }
}

// T = L_i P_{i-1} (rows of L_i sparse), then S_i = D_i - T U_{i-1} with U_{i-1} = K[block i-1,
// block i] given by its rows: S(r, c) -= sum_k T(r, k) U(k, c), k's entries (uidx = c).
__global__ void chain_lp(int bs, const int* lidx, const double* lval, const double* Pprev, double* T) {
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < bs; c += blockDim.x) {
    double s = 0.0;
    for (int e = 0; e < CH_EW; ++e) {
      const int k = lidx[(size_t)r * CH_EW + e];
      if (k >= 0) s = fma(lval[(size_t)r * CH_EW + e], Pprev[(size_t)k * bs + c], s);
    }
    T[(size_t)r * bs + c] = s;
  }
}
// cidx / cval: U_{i-1} by columns (for column c of block i: the rows k of block i-1)
__global__ void chain_schur(int bs, const int* cidx, const double* cval, const double* T, double* S) {
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < bs; c += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < CH_EW; ++e) {
      const int k = cidx[(size_t)c * CH_EW + e];
      if (k >= 0) s = fma(T[(size_t)r * bs + k], cval[(size_t)c * CH_EW + e], s);
    }
    S[(size_t)r * bs + c] -= s;
  }
}

}  // namespace

bool fine_chain_applicable(int n, const int* mp, const int* mi, const int* ap, const int* ai,
                           int* block) {
  const char* env = std::getenv("PE_FINE_CHAIN");
  if (env && std::atoi(env) == 0) return false;
  const bool forced = env && std::atoi(env) != 0;
  if (!forced && n < 16384) return false;
  long long w = 0;
  for (int r = 0; r < n; ++r) {
    for (int t = mp[r]; t < mp[r + 1]; ++t) w = std::max<long long>(w, std::abs(mi[t] - r));
    for (int t = ap[r]; t < ap[r + 1]; ++t) w = std::max<long long>(w, std::abs(ai[t] - r));
  }
  const long long bs = std::max<long long>(64, (w + 63) / 64 * 64);
  if (bs > 512) return false;                  // a ring chunk holds >= 8 rows
  if (!forced && bs * 8 > n) return false;     // not banded enough to pay
  if (block) *block = (int)bs;
  return true;
}

void fine_chain_solve(RefSolveArgs& a) {
  const int n = a.n;
  cudaStream_t st = a.st;
  const double dt = a.t_end / a.n_steps, inv_dt = 1.0 / dt;
  // merged K = M/dt + A rows on the host (sorted, duplicates summed); half-bandwidth
  std::vector<int> kp(n + 1, 0), ki;
  std::vector<double> kv;
  ki.reserve((size_t)a.ap[n] + a.mp[n]);
  kv.reserve((size_t)a.ap[n] + a.mp[n]);
  long long w = 0;
  {
    std::vector<std::pair<int, double>> row;
    for (int r = 0; r < n; ++r) {
      row.clear();
      for (int t = a.mp[r]; t < a.mp[r + 1]; ++t) row.emplace_back(a.mi[t], a.mv[t] * inv_dt);
      for (int t = a.ap[r]; t < a.ap[r + 1]; ++t) row.emplace_back(a.ai[t], a.av[t]);
      std::stable_sort(row.begin(), row.end(),
                       [](const std::pair<int, double>& x, const std::pair<int, double>& y) {
                         return x.first < y.first;
                       });
      for (size_t q = 0; q < row.size(); ++q) {
        if (!ki.empty() && (int)ki.size() > kp[r] && ki.back() == row[q].first) {
          kv.back() += row[q].second;
        } else {
          ki.push_back(row[q].first);
          kv.push_back(row[q].second);
        }
        w = std::max<long long>(w, std::abs(row[q].first - r));
      }
      kp[r + 1] = (int)ki.size();
    }
  }
  const int bs = (int)std::max<long long>(64, (w + 63) / 64 * 64);
  if (bs > 512) throw Error{PE_ERR_ARG, "fine chain solver: half-bandwidth above 512"};
  const int nb = (n + bs - 1) / bs, n_pad = nb * bs, rpc = bs / CH_CS;
  // sparse off-diagonal block rows
  std::vector<int> lidx((size_t)n_pad * CH_EW, -1), uidx((size_t)n_pad * CH_EW, -1);
  std::vector<double> lval((size_t)n_pad * CH_EW, 0.0), uval((size_t)n_pad * CH_EW, 0.0);
  // U blocks by columns (global column c of block i: rows of block i-1), for the Schur update
  std::vector<int> cidx((size_t)n_pad * CH_EW, -1), ccnt(n_pad, 0);
  std::vector<double> cval((size_t)n_pad * CH_EW, 0.0);
  for (int r = 0; r < n; ++r) {
    const int blk = r / bs;
    int nl = 0, nu = 0;
    for (int t = kp[r]; t < kp[r + 1]; ++t) {
      const int cb = ki[t] / bs;
      if (cb == blk) continue;
      if (cb == blk - 1 && nl < CH_EW) {
        lidx[(size_t)r * CH_EW + nl] = ki[t] - cb * bs;
        lval[(size_t)r * CH_EW + nl++] = kv[t];
      } else if (cb == blk + 1 && nu < CH_EW) {
        uidx[(size_t)r * CH_EW + nu] = ki[t] - cb * bs;
        uval[(size_t)r * CH_EW + nu++] = kv[t];
        int& cc = ccnt[ki[t]];
        if (cc >= CH_EW)
          throw Error{PE_ERR_ARG, "fine chain solver: more than " + std::to_string(CH_EW) +
                                      " off-block entries in a column"};
        cidx[(size_t)ki[t] * CH_EW + cc] = r - blk * bs;
        cval[(size_t)ki[t] * CH_EW + cc++] = kv[t];
      } else {
        throw Error{PE_ERR_ARG, "fine chain solver: more than " + std::to_string(CH_EW) +
                                    " off-block entries in a row"};
      }
    }
  }
  Buf<int> d_kp(n + 1), d_ki(ki.size()), d_lidx(lidx.size()), d_uidx(uidx.size()), piv(bs), info(nb);
  Buf<double> d_kv(kv.size()), d_lval(lval.size()), d_uval(uval.size()), d_cval(cval.size());
  Buf<int> d_cidx(cidx.size());
  Buf<double> P((size_t)nb * bs * bs), S((size_t)bs * bs), T((size_t)bs * bs);
  Buf<double> bvec(n), vpad(n_pad);
  Buf<int> d_mp(n + 1), d_mi(a.mp[n]);
  Buf<double> d_mv(a.mp[n]);
  auto up = [&](void* d, const void* h, size_t bytes) {
    if (bytes) PE_CUDA_CHECK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
  };
  up(d_kp.p, kp.data(), sizeof(int) * (n + 1));
  up(d_ki.p, ki.data(), sizeof(int) * ki.size());
  up(d_kv.p, kv.data(), sizeof(double) * kv.size());
  up(d_lidx.p, lidx.data(), sizeof(int) * lidx.size());
  up(d_uidx.p, uidx.data(), sizeof(int) * uidx.size());
  up(d_lval.p, lval.data(), sizeof(double) * lval.size());
  up(d_uval.p, uval.data(), sizeof(double) * uval.size());
  up(d_cidx.p, cidx.data(), sizeof(int) * cidx.size());
  up(d_cval.p, cval.data(), sizeof(double) * cval.size());
  up(bvec.p, a.b, sizeof(double) * n);
  up(d_mp.p, a.mp, sizeof(int) * (n + 1));
  up(d_mi.p, a.mi, sizeof(int) * a.mp[n]);
  up(d_mv.p, a.mv, sizeof(double) * a.mp[n]);
  PE_CUDA_CHECK(cudaMemsetAsync(vpad.p, 0, sizeof(double) * n_pad, st));
  // block factorisation: P_i = (D_i - L_i P_{i-1} U_{i-1})^-1, one after the other
  PE_CUDA_CHECK(cudaMemsetAsync(P.p, 0, sizeof(double) * (size_t)nb * bs * bs, st));
  chain_scatter_diag<<<(n_pad + 255) / 256, 256, 0, st>>>(n, bs, nb, d_kp.p, d_ki.p, d_kv.p, P.p);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  for (int i = 0; i < nb; ++i) {
    double* Di = P.p + (size_t)i * bs * bs;
    // S <- D_i (the LU destroys its input; P_i overwrites D_i)
    PE_CUDA_CHECK(cudaMemcpyAsync(S.p, Di, sizeof(double) * bs * bs, cudaMemcpyDeviceToDevice, st));
    if (i > 0) {
      chain_lp<<<bs, 128, 0, st>>>(bs, d_lidx.p + (size_t)i * bs * CH_EW,
                                   d_lval.p + (size_t)i * bs * CH_EW, Di - (size_t)bs * bs, T.p);
      chain_schur<<<bs, 128, 0, st>>>(bs, d_cidx.p + (size_t)i * bs * CH_EW,
                                      d_cval.p + (size_t)i * bs * CH_EW, T.p, S.p);
      g_launches += 2;
    }
    batched_lu_inverse(bs, 1, S.p, Di, piv.p, info.p + i, st);
  }
  PE_CUDA_CHECK(cudaGetLastError());
  {
    std::vector<int> h(nb);
    PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), info.p, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int i = 0; i < nb; ++i)
      if (h[i] != 0)
        throw Error{PE_ERR_SOLVER, "fine chain solver: singular Schur block " + std::to_string(i)};
  }
  // launch plan
  ChainArgs ca{};
  ca.n = n;
  ca.bs = bs;
  ca.nb = nb;
  ca.rpc = rpc;
  ca.rc = std::min<int>(rpc, std::max<int>(1, (int)(CH_CHUNK / (bs * sizeof(double)))));
  while (rpc % ca.rc) --ca.rc;
  ca.npc = rpc / ca.rc;
  const size_t fixed = sizeof(double) * ((size_t)3 * bs + (size_t)nb * rpc);
  const size_t chunk = sizeof(double) * (size_t)ca.rc * bs;
  const size_t budget = 220 * 1024;
  if (fixed + 2 * chunk > budget)
    throw Error{PE_ERR_ARG, "fine chain solver: problem too large for the cluster's shared memory"};
  ca.stages = (int)std::min<size_t>(8, (budget - fixed) / chunk);
  const size_t smem = fixed + (size_t)ca.stages * chunk;
  ca.P = P.p;
  ca.lidx = d_lidx.p;
  ca.lval = d_lval.p;
  ca.uidx = d_uidx.p;
  ca.uval = d_uval.p;
  ca.v = vpad.p;
  PE_CUDA_CHECK(cudaFuncSetAttribute(fine_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  PE_CUDA_CHECK(cudaFuncSetAttribute(fine_chain_kernel,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CH_CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CH_CS);
  cfg.blockDim = dim3(CH_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;

  const size_t nbytes = (size_t)n * sizeof(double);
  const size_t traj_rows = a.keep ? (size_t)a.n_steps + 1 : 3;
  Buf<double> U(traj_rows * n);
  if (a.u0)
    up(U.p, a.u0, nbytes);
  else
    PE_CUDA_CHECK(cudaMemsetAsync(U.p, 0, nbytes, st));
  struct EventPair {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~EventPair() {
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    }
  } ev;
  if (a.step_ms) {
    PE_CUDA_CHECK(cudaEventCreate(&ev.e0));
    PE_CUDA_CHECK(cudaEventCreate(&ev.e1));
    PE_CUDA_CHECK(cudaEventRecord(ev.e0, st));
  }
  for (int s = 0; s < a.n_steps; ++s) {
    const double* src = U.p + (size_t)(a.keep || s == 0 ? s : 1 + ((s - 1) & 1)) * n;
    ca.x = U.p + (size_t)(a.keep ? s + 1 : 1 + (s & 1)) * n;
    fine_rhs(n, d_mp.p, d_mi.p, d_mv.p, inv_dt, src, bvec.p, vpad.p, st);
    PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fine_chain_kernel, ca));
    g_launches += 2;
  }
  PE_CUDA_CHECK(cudaGetLastError());
  if (a.step_ms) {
    PE_CUDA_CHECK(cudaEventRecord(ev.e1, st));
    PE_CUDA_CHECK(cudaEventSynchronize(ev.e1));
    PE_CUDA_CHECK(cudaEventElapsedTime(a.step_ms, ev.e0, ev.e1));
  }
  if (a.keep) {
    PE_CUDA_CHECK(cudaMemcpyAsync(a.states_h, U.p, nbytes * traj_rows, cudaMemcpyDeviceToHost, st));
  } else {
    PE_CUDA_CHECK(cudaMemcpyAsync(a.states_h, U.p, nbytes, cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaMemcpyAsync(a.states_h + n, U.p + (size_t)(1 + ((a.n_steps - 1) & 1)) * n, nbytes,
                                  cudaMemcpyDeviceToHost, st));
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace pe
