// libpe context: device-resident operators, factor caches and work buffers.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <map>
#include <vector>

#include "pe_internal.h"

namespace pe {

// Owning device buffer (bytes); grows, never shrinks.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (n == 0) return;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error{PE_ERR_NOMEM, "cudaMalloc of " + std::to_string(n) + " bytes failed"};
    }
    bytes = n;
  }
  double* d() const { return static_cast<double*>(p); }
  int* i() const { return static_cast<int*>(p); }
};

// One WR sweep captured as a CUDA graph per counter parity; `key` records every pointer
// and size baked into the nodes, so any reallocation or re-setup forces a recapture.
struct SweepGraphs {
  std::vector<const void*> key;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  cudaGraphExec_t loop = nullptr;  // whole WR solve: one while-node around one sweep
  int kernels = 0;  // kernel launches recorded per captured sweep
};

struct FineStats {
  double gemm_flops = 0;   // algorithmic flops issued by the GEMM kernels of the last fine call
  double gemm_ms = 0;      // summed CUDA-event time of those launches (profiling mode only)
  double other_ms = 0;     // summed time of the sweep's non-DMMA kernels (scans, decide)
  int launches = 0;
};

}  // namespace pe

struct pe_ctx {
  int E = 0, d1 = 0, d2 = 0, d = 0, maxc = 0, J = 0, device = 0;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cudaStream_t setup_stream = nullptr;

  // reduced system, row-major, member-strided
  pe::DevBuf M11, A11, M12, A12, M22, A22, f1, f2;
  std::vector<char> member_set;

  // sequential fine: X_{s+1} = T [X_s; D_s] + cvec   (T: E x d x 2d); cvec = Lf [f1; f2]
  double seq_dt = -1.0;
  pe::DevBuf T, cvec, Lf;
  // coarse: G(x) = Phi x + gG                         (Phi: E x d x d); gG = LG [f1; f2]
  double coarse_dt = -1.0;
  pe::DevBuf Phi, gG, LG;
  // time-dependent loads: per-call load-term series (sequential bias, WR rhs / h terms,
  // coarse terms) and their permuted inputs
  pe::DevBuf LB, LF1, LF2, LB1, LB2, LGs;
  // all-at-once
  bool wr_ready = false;
  double wr_dt = 0, wr_alpha = 0, wr_tol = 0;
  int wr_max_iter = 0;
  int wr_last_nc = 0;          // intervals of the last fine_allatonce (Ux_cur / Wx_cur hold them)
  bool wr_last_loads = false;  // ... and whether it ran with time-dependent loads (LF1 rows)
  int wr_nk = 0;  // solved time modes (half spectrum, floor(J/2) + 1)
  pe::DevBuf Bk, BkT, RW, M11dt, GW, cg, Emat, Finv, Fw;
  // modal w recursion (setup_modal): E = Vm diag(lam) Vinv; GZ = Vinv GW, cgz = Vinv cg
  bool wr_modal = false;   // decided by setup (every member passed the reconstruction check)
  bool use_modal = true;   // user switch (pe_set_modal)
  pe::DevBuf Vm, Vinv, lam, GZ, cgz, Z0, Hz;
  // full modal sweep (setup_modal_full, wr_modal.cu): both pencils diagonalised
  bool wr_modal_full = false;
  bool wr_modal_avail = false;  // modal operators built (also when the tiny kernel is used)
  pe::DevBuf Vcat, Vicat, Ucat, RT, GT, f1t, cgt, acoef, cden;
  pe::DevBuf Yb[2], Zb[2], DYm, EYZ, Y0m, nrmp, colmax;

  // work buffers
  pe::DevBuf Xin, Xout, Xa, Xb, Da, Db, Xs, Zg, gcnt, wticket;
  pe::DevBuf Ux_cur, Ux_new, Wx_cur, Wx_new, R, P, Q, DU, DW, V, colstate, counter;
  pe::DevBuf partial, diff, Gc, active, hist_tmp, nrm, rhist, splitws;
  cudaStream_t work = nullptr;           // capture stream for the sweep graphs
  bool use_graphs = true;
  bool device_loop = true;  // WR sweep loop as a conditional while-node (modal path)
  int graph_kernels = 0;   // kernels per captured sweep (launch accounting)
  std::map<int, pe::SweepGraphs> sweep_graphs;  // keyed by interval count
  int* pinned_count = nullptr;
  double* pinned_diff = nullptr;
  size_t pinned_diff_n = 0;

  long long launches_at_create = 0;
  cudaEvent_t ev_mid = nullptr;  // fine/coarse boundary inside pe_parareal_run
  bool profiling = false;
  bool use_recur = true;  // persistent cluster recurrences (else one GEMM per step)
  std::vector<cudaEvent_t> prof_events;
  std::vector<char> prof_dmma;  // per timed launch: DMMA-class (1) or other (0)
  int prof_used = 0;
  pe::FineStats stats;
};
