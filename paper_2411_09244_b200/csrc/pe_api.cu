// C ABI of libpe (include/pe.h): context, uploads, fine propagators, fused coarse
// correction and the device-resident parareal loop.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pe.h"
#include "pe_ctx.h"

namespace pe {

long long g_launches = 0;
bool g_pdl = getenv("PE_NO_PDL") == nullptr;
static thread_local std::string t_err;
void set_error(const std::string& m) { t_err = m; }

void setup_sequential(pe_ctx* c, double dt);
void setup_coarse(pe_ctx* c, double dt);
void setup_allatonce(pe_ctx* c, double dt, double alpha, double tol, int max_iter);

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return PE_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PE_ERR_CUDA;
  } catch (...) {
    set_error("unknown error");
    return PE_ERR_CUDA;
  }
}

static void require(bool ok, int code, const char* msg) {
  if (!ok) throw Error{code, msg};
}

static void bind(pe_ctx* c) { PE_CUDA_CHECK(cudaSetDevice(c->device)); }

// Graph-cache key entry for a double baked into captured kernel arguments: the exact IEEE
// bit pattern, so any change of alpha / tol / dt (however small) forces a recapture.
static const void* dkey(double v) {
  uint64_t u;
  std::memcpy(&u, &v, sizeof u);
  return (const void*)(uintptr_t)u;
}

// Split-K workspace: partial planes + per-tile tickets that must start (and are left) zero.
static void ensure_zeroed(DevBuf& b, size_t bytes) {
  if (bytes <= b.bytes) return;
  b.ensure(bytes);
  PE_CUDA_CHECK(cudaMemset(b.p, 0, b.bytes));
}

// Launch `fn` (one DMMA-class kernel doing `flops` algorithmic flops) with optional
// per-launch CUDA-event timing (bench roofline pass).
template <class F>
static void timed(pe_ctx* c, bool dmma, cudaStream_t st, F&& fn) {
  if (c->profiling) {
    if ((int)c->prof_events.size() < 2 * (c->prof_used + 1)) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        PE_CUDA_CHECK(cudaEventCreate(&e));
        c->prof_events.push_back(e);
      }
    }
    if ((int)c->prof_dmma.size() < c->prof_used + 1) c->prof_dmma.resize(c->prof_used + 64);
    c->prof_dmma[c->prof_used] = dmma ? 1 : 0;
    PE_CUDA_CHECK(cudaEventRecord(c->prof_events[2 * c->prof_used], st));
    fn();
    PE_CUDA_CHECK(cudaEventRecord(c->prof_events[2 * c->prof_used + 1], st));
    ++c->prof_used;
  } else {
    fn();
  }
}
template <class F>
static void profiled(pe_ctx* c, double flops, cudaStream_t st, F&& fn) {
  timed(c, true, st, fn);
  c->stats.gemm_flops += flops;
  c->stats.launches += 1;
}
// a non-DMMA kernel of the fine sweep (scans, decide): timed separately in profiling mode
template <class F>
static void profiled_other(pe_ctx* c, cudaStream_t st, F&& fn) {
  timed(c, false, st, fn);
}

static void run_gemm(pe_ctx* c, const GemmParams& p, cudaStream_t st) {
  profiled(c, gemm_flops(p), st, [&] { gemm_f64(p, st); });
}

static void collect_profile(pe_ctx* c, cudaStream_t st) {
  if (!c->profiling || c->prof_used == 0) return;
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  for (int i = 0; i < c->prof_used; ++i) {
    float ms = 0;
    PE_CUDA_CHECK(cudaEventElapsedTime(&ms, c->prof_events[2 * i], c->prof_events[2 * i + 1]));
    (c->prof_dmma[i] ? c->stats.gemm_ms : c->stats.other_ms) += ms;
  }
  c->prof_used = 0;
}

// ------------------------------------------------------------------ sequential fine
// X_in/X_out: (E, nc, d) == per member a column-major d x nc matrix.
// With X_prev == nullptr the lags are reset (D_0 = 0, interval start); otherwise
// D_0 = X_in - X_prev (a single split_step with explicit lags, stepping.py:122-147).
// ------------------------------------------------------------------ time-dependent loads
// The reference evaluates loads at each step's end time (stepping.py:125,164;
// allatonce.py:212-218).  A call with a load series F (E, nc, J, d) -- [f1(t); f2(t)] per
// (member, interval column, substep) -- turns the constant bias vectors into per-column
// terms: the sequential step's Lf F (Lf from setup_sequential), the WR rhs term V1^T F1 and
// h term dt V2^T F2, the coarse step's K_G^-1 F.
__global__ void k_perm_seni(long long E, int nc, int J, int d, int k0, int dk,
                            const double* __restrict__ src, double* __restrict__ dst,
                            int step_major) {
  // src [e][n][s][k] (row length d) -> dst rows of dk: step_major ? [s][e][n] : [e][s][n]
  const long long total = E * nc * J * (long long)dk;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(q % dk);
    long long r = q / dk;
    const int s = (int)(r % J);
    r /= J;
    const int n = (int)(r % nc);
    const long long e = r / nc;
    const long long o = step_major ? (((long long)s * E + e) * nc + n) * dk + k
                                   : ((e * J + s) * nc + n) * dk + k;
    dst[o] = src[q / dk * d + k0 + k];
  }
}

static int loads_grid(long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 16));
}

// LB [s][e][n][d] = Lf F (the sequential step's per-column bias series)
static double* seq_load_terms(pe_ctx* c, int nc, int J, const double* F, cudaStream_t st) {
  const int d = c->d, E = c->E;
  const size_t n = (size_t)E * nc * J * d;
  c->LF1.ensure(sizeof(double) * n + 8);
  c->LB.ensure(sizeof(double) * n + 8);
  GemmParams p;  // tmp (E, nc, J, d) = Lf F, columns (n, s) contiguous
  p.M = d;
  p.N = nc * J;
  p.nb1 = E;
  p.nseg = 1;
  p.seg[0].A = Operand{c->Lf.d(), d, 1, (long long)d * d, 0};
  p.seg[0].B = Operand{F, 1, d, (long long)nc * J * d, 0};
  p.seg[0].K = d;
  p.C = c->LF1.d();
  p.c_i = 1;
  p.c_j = d;
  p.c_b1 = (long long)nc * J * d;
  run_gemm(c, p, st);
  k_perm_seni<<<loads_grid((long long)n), 256, 0, st>>>(E, nc, J, d, 0, d, c->LF1.d(), c->LB.d(), 1);
  ++g_launches;
  PE_CUDA_CHECK(cudaGetLastError());
  return c->LB.d();
}

// LGs (E, N, d) = K_G^-1 Fc  (the coarse step's per-interval load terms)
static double* coarse_load_terms(pe_ctx* c, int N, const double* Fc, cudaStream_t st) {
  const int d = c->d, E = c->E;
  c->LGs.ensure(sizeof(double) * (size_t)E * N * d + 8);
  GemmParams p;
  p.M = d;
  p.N = N;
  p.nb1 = E;
  p.nseg = 1;
  p.seg[0].A = Operand{c->LG.d(), d, 1, (long long)d * d, 0};
  p.seg[0].B = Operand{Fc, 1, d, (long long)N * d, 0};
  p.seg[0].K = d;
  p.C = c->LGs.d();
  p.c_i = 1;
  p.c_j = d;
  p.c_b1 = (long long)N * d;
  run_gemm(c, p, st);
  return c->LGs.d();
}

static void fine_sequential(pe_ctx* c, const double* X_in, double* X_out, int nc,
                            cudaStream_t st, const double* X_prev = nullptr, int steps = -1,
                            const double* Fload = nullptr, const int* active = nullptr) {
  const int d = c->d, E = c->E, J = steps < 0 ? c->J : steps;
  // time-dependent loads: per-(step, column) bias terms, per-step GEMMs only
  const double* LB = Fload ? seq_load_terms(c, nc, J, Fload, st) : nullptr;
  const size_t n = (size_t)E * nc * d;
  c->Xa.ensure(sizeof(double) * n + 8);
  c->Xb.ensure(sizeof(double) * n + 8);
  c->Da.ensure(sizeof(double) * n + 8);
  c->Db.ensure(sizeof(double) * n + 8);
  ensure_zeroed(c->splitws, sizeof(double) * (8 * n + 32768));
  c->stats = FineStats();
  const double* Xs = X_in;
  const double* Ds = nullptr;  // D_0 = 0 at the interval start (lags reset, stepping.py:180)
  double* bufX[2] = {c->Xa.d(), c->Xb.d()};
  double* bufD[2] = {c->Da.d(), c->Db.d()};
  if (X_prev) {
    c->Xin.ensure(sizeof(double) * n + 8);
    sub((long long)n, X_in, X_prev, c->Xin.d(), st);
    Ds = c->Xin.d();
  } else if (!LB) {
    int rpc_, cs_;
    size_t sm_;
    // algorithmic flops of J split steps: u rows contract [X; Dw], w rows [X; Dw; Du]
    const double chain_flops = 2.0 * nc * E * J * ((double)c->d1 * (d + c->d2) + (double)c->d2 * 2 * d);
    if (J > 0 && c->use_recur && recur_plan(d, 2 * d, &rpc_, &cs_, &sm_)) {
      // all J substeps in one persistent cluster launch (T's row slices fit in smem)
      c->Xs.ensure(sizeof(double) * 4 * n + 8);
      profiled(c, chain_flops, st, [&] {
        recur_seq(E, d, nc, J, c->T.d(), c->cvec.d(), X_in, X_out, c->Xs.d(), st);
      });
      collect_profile(c, st);
      return;
    }
    if (J > 0 && c->use_recur && seqgrid_fits(E, c->d1, c->d2, nc)) {
      // T too large for a cluster: all SMs, T row slices resident, state through L2
      c->Zg.ensure(sizeof(double) * 2 * (size_t)nc * 2 * d + 16);
      c->gcnt.ensure(sizeof(unsigned) * ((size_t)nc + 8));
      profiled(c, chain_flops, st, [&] {
        seqgrid_seq(c->d1, c->d2, nc, J, c->T.d(), c->cvec.d(), X_in, X_out, c->Zg.d(),
                    (unsigned*)c->gcnt.p, st);
      });
      collect_profile(c, st);
      return;
    }
  }
  // Ensembles whose operators exceed L2 (cfg4: 64 x 5.8 MB) run member chunks through all
  // J steps, so a chunk's T stays L2-resident across its steps instead of streaming every
  // member's T from HBM once per step.  Members are independent: same arithmetic.
  static const int chunk_env = getenv("PE_SEQ_CHUNK") ? atoi(getenv("PE_SEQ_CHUNK")) : 0;
  // measured at cfg4 (E = 64, d = 600, tools/chunk_sweep.sh, TMA 128x32 tiles): one chunk
  // of 64 members 7.06 ms, 2 x 32 7.25 ms, 3 x 22 10.0 ms, 4 x 16 12.7 ms (smaller chunks
  // underfill the SMs); larger ensembles run in chunks of 64
  int EC = chunk_env > 0 ? chunk_env : 64;
  if (EC >= E || J < 2) EC = E;
  const long long xs = (long long)nc * d;
  const double* X0 = Xs;
  const double* D0 = Ds;
  for (int e0 = 0; e0 < E; e0 += EC) {
    const int ec = std::min(EC, E - e0);
    const long long xo = e0 * xs;
    Xs = X0 + xo;
    Ds = D0 ? D0 + xo : nullptr;
    if (!LB && J >= 2) {
      // ensembles: all J steps in one cooperative row-balanced launch (per-member counters
      // order the steps; T streams on across the step boundaries)
      GemmParams p2;
      p2.M = d;
      p2.N = nc;
      p2.nb1 = ec;
      p2.nseg = 2;
      p2.seg[0].A = Operand{c->T.d() + e0 * 2LL * d * d, 2LL * d, 1, 2LL * d * d, 0};
      p2.seg[0].B = Operand{Xs, 1, d, xs, 0};
      p2.seg[0].K = d;
      p2.seg[1].A = Operand{c->T.d() + e0 * 2LL * d * d + d, 2LL * d, 1, 2LL * d * d, 0};
      p2.seg[1].B = Operand{bufD[0] + xo, 1, d, xs, 0};
      p2.seg[1].K = d;
      p2.C = bufX[0] + xo;
      p2.c_i = 1;
      p2.c_j = d;
      p2.c_b1 = xs;
      p2.bias = c->cvec.d() + (long long)e0 * d;
      p2.bias_b1 = d;
      if (gemm_rowbalanced_chain_eligible(p2, c->d1, 0, c->d1)) {
        double* bx[2] = {bufX[0] + xo, bufX[1] + xo};
        double* bd[2] = {bufD[0] + xo, bufD[1] + xo};
        c->gcnt.ensure(sizeof(unsigned) * ((size_t)ec + 8));
        // algorithmic flops: the u x Du block is a structural zero; D_0 = 0 has no product
        const double per2 = 2.0 * ec * nc * ((double)d * 2 * d - (double)c->d1 * c->d1);
        const double per1 = 2.0 * ec * nc * (double)d * d;
        const double flops = (Ds ? per2 : per1) + (J - 1) * per2;
        profiled(c, flops, st, [&] {
          gemm_f64_rowbalanced_chain(p2, c->d1, 0, c->d1, J, Xs, Ds, bx, bd, X_out + xo,
                                     (unsigned*)c->gcnt.p, active ? active + e0 : nullptr, st);
        });
        continue;
      }
    }
    for (int s = 0; s < J; ++s) {
      const bool last = (s == J - 1);
      double* Xn = (last ? X_out : bufX[s & 1]) + xo;
      double* Dn = last ? nullptr : bufD[s & 1] + xo;
      GemmParams p;
      p.M = d;
      p.N = nc;
      p.nb1 = ec;
      p.nseg = Ds ? 2 : 1;
      p.seg[0].A = Operand{c->T.d() + e0 * 2LL * d * d, 2LL * d, 1, 2LL * d * d, 0};
      p.seg[0].B = Operand{Xs, 1, d, xs, 0};
      p.seg[0].K = d;
      if (Ds) {
        p.seg[1].A = Operand{c->T.d() + e0 * 2LL * d * d + d, 2LL * d, 1, 2LL * d * d, 0};
        p.seg[1].B = Operand{Ds, 1, d, xs, 0};
        p.seg[1].K = d;
      }
      p.C = Xn;
      p.c_i = 1;
      p.c_j = d;
      p.c_b1 = xs;
      p.ws = c->splitws.d();
      p.ws_doubles = c->splitws.bytes / sizeof(double);
      p.bias = c->cvec.d() + (long long)e0 * d;
      p.bias_b1 = d;
      if (LB) {  // C = T [X; D] + LB[s]  (per-column load terms replace the bias)
        p.bias = nullptr;
        p.Cin = LB + ((size_t)s * E + e0) * (size_t)nc * d;
        p.beta = 1.0;
      }
      if (Dn) {
        p.D = Dn;
        p.Xp = Xs;
      }
      // ensembles: one row-balanced persistent launch per step, skipping T's exact-zero
      // u x Du block (rows < d1, D-segment columns < d1); else the tiled kernels
      if (gemm_rowbalanced_eligible(p, Ds ? c->d1 : 0, 0, Ds ? c->d1 : 0)) {
        // algorithmic flops: the skipped u x Du block is a structural zero
        const double zero = Ds ? 2.0 * ec * nc * (double)c->d1 * c->d1 : 0.0;
        profiled(c, gemm_flops(p) - zero, st, [&] {
          gemm_f64_rowbalanced(p, Ds ? c->d1 : 0, 0, Ds ? c->d1 : 0, st);
        });
      } else {
        run_gemm(c, p, st);
      }
      Xs = Xn;
      Ds = Dn;
    }
  }
  if (J == 0) PE_CUDA_CHECK(cudaMemcpyAsync(X_out, X_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  collect_profile(c, st);
}

// ------------------------------------------------------------------ all-at-once fine
// Replays one captured sweep graph per buffer parity (or launches `body` directly), with
// the pipelined host loop: sweep i+1 is enqueued before the host reads sweep i's
// active-interval count, so the device never waits on the host; the extra sweep after the
// last interval stopped is fully masked.  `key` lists every pointer / value baked into the
// nodes, so any reallocation or re-setup forces a recapture.
//
// Device loop (`loop_ok`: the body takes the conditional handle, modal path): the whole
// solve is ONE graph launch, a conditional while-node around one captured sweep whose
// decide kernel sets the condition to "some interval still iterating" -- no host round trip
// per sweep and no speculative sweep after the last one.  Falls back to the pipelined host
// loop if the driver rejects the conditional graph.
template <class Body>
static void run_sweeps(pe_ctx* c, int nc, int max_iter, const std::vector<const void*>& key,
                       Body&& body, cudaStream_t st, bool loop_ok = false,
                       const int* dev_sweeps = nullptr) {
  int* host_cnt = c->pinned_count;
  static const bool no_graphs = getenv("PE_NO_GRAPHS") != nullptr;
  static const bool no_loop = getenv("PE_NO_DEVICE_LOOP") != nullptr;
  const bool graphs = c->use_graphs && !c->profiling && !no_graphs &&
                      getenv("PE_RECUR_TRACE") == nullptr;
  SweepGraphs* sg = nullptr;
  if (graphs && loop_ok && c->device_loop && !no_loop) {
    sg = &c->sweep_graphs[nc];
    if (sg->key != key || !sg->loop) {
      for (auto& ex : sg->exec)
        if (ex) {
          cudaGraphExecDestroy(ex);
          ex = nullptr;
        }
      if (sg->loop) {
        cudaGraphExecDestroy(sg->loop);
        sg->loop = nullptr;
      }
      const long long launches_before = g_launches;
      bool ok = true;
      cudaGraph_t g = nullptr;
      try {
        PE_CUDA_CHECK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        PE_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        PE_CUDA_CHECK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t bg = cp.conditional.phGraph_out[0];
        PE_CUDA_CHECK(cudaStreamBeginCaptureToGraph(c->work, bg, nullptr, nullptr, 0,
                                                    cudaStreamCaptureModeThreadLocal));
        try {
          body(0, c->work, h, 1);
        } catch (...) {
          cudaStreamEndCapture(c->work, &bg);
          throw;
        }
        PE_CUDA_CHECK(cudaStreamEndCapture(c->work, &bg));
        PE_CUDA_CHECK(cudaGraphInstantiate(&sg->loop, g, 0));
      } catch (const Error&) {
        ok = false;
        cudaGetLastError();
        if (sg->loop) cudaGraphExecDestroy(sg->loop);
        sg->loop = nullptr;
      }
      if (g) cudaGraphDestroy(g);
      sg->kernels = (int)(g_launches - launches_before);
      g_launches = launches_before;
      if (!ok) {
        c->device_loop = false;  // this driver rejects it: pipelined host loop from now on
        sg->key.clear();
        run_sweeps(c, nc, max_iter, key, body, st, false, nullptr);
        return;
      }
      sg->key = key;
    }
    PE_CUDA_CHECK(cudaGraphLaunch(sg->loop, st));
    if (dev_sweeps) {  // launch evidence: kernels per sweep x sweeps run
      PE_CUDA_CHECK(cudaMemcpyAsync(host_cnt, dev_sweeps, sizeof(int), cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      g_launches += (long long)sg->kernels * host_cnt[0];
    } else {
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    return;
  }
  if (graphs) {
    sg = &c->sweep_graphs[nc];
    if (sg->key != key || sg->loop) {
      for (auto& ex : sg->exec)
        if (ex) {
          cudaGraphExecDestroy(ex);
          ex = nullptr;
        }
      if (sg->loop) {
        cudaGraphExecDestroy(sg->loop);
        sg->loop = nullptr;
      }
      const long long launches_before = g_launches;  // capture launches nothing
      for (int par = 0; par < 2; ++par) {
        cudaGraph_t g;
        PE_CUDA_CHECK(cudaStreamBeginCapture(c->work, cudaStreamCaptureModeThreadLocal));
        try {
          body(par, c->work, cudaGraphConditionalHandle(0), 0);
        } catch (...) {
          cudaStreamEndCapture(c->work, &g);
          throw;
        }
        PE_CUDA_CHECK(cudaStreamEndCapture(c->work, &g));
        PE_CUDA_CHECK(cudaGraphInstantiate(&sg->exec[par], g, 0));
        PE_CUDA_CHECK(cudaGraphDestroy(g));
      }
      sg->key = key;
      sg->kernels = (int)((g_launches - launches_before) / 2);  // kernel nodes per graph
      g_launches = launches_before;
    }
  }
  cudaEvent_t ev[2];
  PE_CUDA_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  PE_CUDA_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto enqueue_sweep = [&](int sweep) {
    if (sg) {
      PE_CUDA_CHECK(cudaGraphLaunch(sg->exec[sweep & 1], st));
      g_launches += c->graph_kernels;
    } else {
      body(sweep & 1, st, cudaGraphConditionalHandle(0), 0);
    }
    PE_CUDA_CHECK(cudaEventRecord(ev[sweep & 1], st));
    collect_profile(c, st);
  };
  if (sg) c->graph_kernels = sg->kernels;  // kernels per graph replay (launch evidence)
  enqueue_sweep(0);
  for (int sweep = 1; sweep <= max_iter; ++sweep) {
    if (sweep < max_iter) enqueue_sweep(sweep);
    PE_CUDA_CHECK(cudaEventSynchronize(ev[(sweep - 1) & 1]));
    if (host_cnt[(sweep - 1) & 1] == 0) break;
  }
  PE_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
}

// The modal sweep (wr_modal.cu; setup_modal_full): per sweep the rhs GEMM, the u scan, the
// g GEMM, the w scan, the residual-norm GEMM(s) and the stop decision.
static void fine_allatonce_modal(pe_ctx* c, const double* X_in, double* X_out, int nc,
                                 int* sweeps, int* reasons, double* resid_hist, cudaStream_t st,
                                 const double* Fload = nullptr) {
  const int d1 = c->d1, d2 = c->d2, d = c->d, E = c->E, J = c->J;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const double alpha = c->wr_alpha, tol = c->wr_tol, dt = c->wr_dt;
  const int max_iter = c->wr_max_iter;
  const long long vstride = (long long)d1 * d1 + (long long)d2 * d2;
  const long long NJ = (long long)J * nc;
  const int g1 = (d1 + 7) / 8, g2 = (d2 + 7) / 8;
  // one waveform buffer per block, updated in place by the scans (each thread reads an
  // element before it overwrites it; stopped intervals are skipped, so they keep the
  // waveforms of their last sweep without any commit copy)
  // working set per sweep: h reuses r~'s buffer (r~ is dead once the u scan has read it)
  // and dY shares e_Z's (dY is dead once the h GEMM has read it; the w scan writes e_Z
  // afterwards).  The six sweep arrays are one arena (~60 MB at cfg2).
  const long long Lm = std::max(L1, L2);
  auto al = [](long long n) { return (n + 31) & ~31LL; };  // 256-byte aligned sub-arrays
  const long long nEY = al(E * J * L1), nEZ = al(E * J * Lm), nR = al(E * J * Lm),
                  nDZ = al(E * J * L2), nY = al(E * (J + 2) * L1), nZ = al(E * (J + 2) * L2);
  const size_t arena_bytes = sizeof(double) * (size_t)(nEY + nEZ + nR + nDZ + nY + nZ) + 256;
  c->EYZ.ensure(arena_bytes);
  double* EY = c->EYZ.d();
  double* EZ = EY + nEY;
  double* Rb = EZ + nEZ;  // r~, then h
  double* DZ = Rb + nR;
  double* Yw = DZ + nDZ;
  double* Zw = Yw + nY;
  double* DYb = EZ;  // dY, then e_Z
  c->Y0m.ensure(sizeof(double) * E * L1 + 8);
  c->Z0.ensure(sizeof(double) * E * L2 + 8);
  c->nrmp.ensure(sizeof(double) * (size_t)(g1 + g2) * E * NJ + 8);
  c->Ux_cur.ensure(sizeof(double) * E * (J + 2) * L1 + 8);
  c->Ux_new.ensure(sizeof(double) * E * (J + 2) * L1 + 8);
  c->Wx_cur.ensure(sizeof(double) * E * (J + 2) * L2 + 8);
  c->Wx_new.ensure(sizeof(double) * E * (J + 2) * L2 + 8);
  c->colstate.ensure(sizeof(WrColumnState) * E * nc + 8);
  c->rhist.ensure(sizeof(double) * (size_t)E * nc * max_iter + 8);
  c->counter.ensure(sizeof(int) * 4);
  ensure_zeroed(c->wticket, sizeof(unsigned) * (size_t)E * nc + 8);  // self-resetting ticket
  c->colmax.ensure(sizeof(unsigned long long) * 2 * (size_t)E * nc + 8);
  PE_CUDA_CHECK(cudaMemsetAsync(c->colmax.p, 0, c->colmax.bytes, st));
  c->stats = FineStats();
  WrColumnState* cs = (WrColumnState*)c->colstate.p;
  int* cnt = c->counter.i();

  // seeds: y0 = V1^-1 u0, z0 = V2^-1 w0 (X_in: (E, nc, d))
  wr_state_init((long long)E * nc, cs, c->rhist.d(), max_iter, st);
  auto basis_gemm = [&](int M, const double* A, const double* B, long long b_j, long long b_b,
                        double* C, long long c_b, int ncols) {
    GemmParams p;
    p.M = M;
    p.N = ncols;
    p.nb1 = E;
    p.nseg = 1;
    p.seg[0].A = Operand{A, M, 1, vstride, 0};
    p.seg[0].B = Operand{B, 1, b_j, b_b, 0};
    p.seg[0].K = M;
    p.C = C;
    p.c_i = 1;
    p.c_j = M;
    p.c_b1 = c_b;
    gemm_f64(p, st);
  };
  basis_gemm(d1, c->Vicat.d(), X_in, d, (long long)nc * d, c->Y0m.d(), L1, nc);
  basis_gemm(d2, c->Vicat.d() + (long long)d1 * d1, X_in + d1, d, (long long)nc * d, c->Z0.d(), L2, nc);
  modal_seed(E, nc, d1, d2, J, c->Y0m.d(), c->Z0.d(), Yw, nullptr, Zw, nullptr, DZ, st);

  // time-dependent loads: per-(substep, interval) rhs / h load terms replace V1^T f1 and
  // dt V2^T f2 (allatonce.py:212-218 load rows; build_rhs :156, _w_sweep :224)
  const double* LB1 = nullptr;
  const double* LB2 = nullptr;
  if (Fload) {
    const size_t n1 = (size_t)E * NJ * d1, n2 = (size_t)E * NJ * d2;
    c->LF1.ensure(sizeof(double) * n1 + 8);
    c->LF2.ensure(sizeof(double) * n2 + 8);
    c->LB1.ensure(sizeof(double) * n1 + 8);
    c->LB2.ensure(sizeof(double) * n2 + 8);
    k_perm_seni<<<loads_grid((long long)n1), 256, 0, st>>>(E, nc, J, d, 0, d1, Fload, c->LF1.d(), 0);
    k_perm_seni<<<loads_grid((long long)n2), 256, 0, st>>>(E, nc, J, d, d1, d2, Fload, c->LF2.d(), 0);
    g_launches += 2;
    PE_CUDA_CHECK(cudaGetLastError());
    auto tgemm = [&](int M, const double* V, const double* B, double* C, double alpha_) {
      GemmParams p;  // C = alpha V^T B over all (s, n) columns, V row-major M x M
      p.M = M;
      p.N = (int)NJ;
      p.nb1 = E;
      p.nseg = 1;
      p.alpha = alpha_;
      p.seg[0].A = Operand{V, 1, M, vstride, 0};
      p.seg[0].B = Operand{B, 1, M, NJ * M, 0};
      p.seg[0].K = M;
      p.C = C;
      p.c_i = 1;
      p.c_j = M;
      p.c_b1 = NJ * M;
      run_gemm(c, p, st);
    };
    tgemm(d1, c->Vcat.d(), c->LF1.d(), c->LB1.d(), 1.0);
    tgemm(d2, c->Vcat.d() + (long long)d1 * d1, c->LF2.d(), c->LB2.d(), dt);
    LB1 = c->LB1.d();
    LB2 = c->LB2.d();
  }
  // loop-invariant GEMM parameter blocks (buffer parity fills in the B / C pointers)
  auto rhs_params = [&](const double* Zcur) {
    GemmParams r;  // r~ = [A~ | M~][Z_s; DZ_s] + V1^T f1   (build_rhs, allatonce.py:136-158)
    r.M = d1;
    r.N = (int)NJ;
    r.nb1 = E;
    r.nseg = 2;
    r.seg[0].A = Operand{c->RT.d(), 2LL * d2, 1, 2LL * d1 * d2, 0};
    r.seg[0].B = Operand{Zcur + L2, 1, d2, (J + 2) * L2, 0};
    r.seg[0].K = d2;
    r.seg[1].A = Operand{c->RT.d() + d2, 2LL * d2, 1, 2LL * d1 * d2, 0};
    r.seg[1].B = Operand{DZ, 1, d2, J * L2, 0};
    r.seg[1].K = d2;
    r.C = Rb;
    r.c_i = 1;
    r.c_j = d1;
    r.c_b1 = J * L1;
    r.bias = c->f1t.d();
    r.bias_b1 = d1;
    if (LB1) {
      r.bias = nullptr;
      r.Cin = LB1;
      r.beta = 1.0;
    }
    return r;
  };
  auto g_params = [&](const double* Ynew) {
    GemmParams g;  // h = [G~u | G~d][Y_s; DY_s] + dt V2^T f2   (_w_sweep, allatonce.py:220-224)
    g.M = d2;
    g.N = (int)NJ;
    g.nb1 = E;
    g.nseg = 2;
    g.seg[0].A = Operand{c->GT.d(), 2LL * d1, 1, 2LL * d1 * d2, 0};
    g.seg[0].B = Operand{Ynew + 2 * L1, 1, d1, (J + 2) * L1, 0};
    g.seg[0].K = d1;
    g.seg[1].A = Operand{c->GT.d() + d1, 2LL * d1, 1, 2LL * d1 * d2, 0};
    g.seg[1].B = Operand{DYb, 1, d1, J * L1, 0};
    g.seg[1].K = d1;
    g.C = Rb;
    g.c_i = 1;
    g.c_j = d2;
    g.c_b1 = J * L2;
    g.bias = c->cgt.d();
    g.bias_b1 = d2;
    if (LB2) {
      g.bias = nullptr;
      g.Cin = LB2;
      g.beta = 1.0;
    }
    return g;
  };
  // residual norms ||V1 EY_s|| = ||U1 EY_s|| (U1 upper-triangular, setup.cu norm_factor),
  // likewise W, per (s, interval) as 8-row block partials
  std::vector<GemmParams> norms;
  long long nu_g, nu_m, nw_g, nw_m;
  const double *nu, *nw;
  if (d1 == d2) {  // one launch, the two sides as the inner batch level
    GemmParams q;
    q.M = d1;
    q.N = (int)NJ;
    q.nb1 = E;
    q.nb2 = 2;
    q.nseg = 1;
    q.seg[0].A = Operand{c->Ucat.d(), d1, 1, vstride, (long long)d1 * d1};
    q.seg[0].B = Operand{EY, 1, d1, J * L1, E * J * L1};
    q.seg[0].K = d1;
    q.tri_upper = 1;
    q.nrm = c->nrmp.d();
    q.nrm_ld = 2LL * E * NJ;
    norms.push_back(q);
    nu = c->nrmp.d();
    nw = c->nrmp.d() + NJ;
    nu_g = nw_g = 2LL * E * NJ;
    nu_m = nw_m = 2 * NJ;
  } else {
    for (int side = 0; side < 2; ++side) {
      const int M = side ? d2 : d1;
      GemmParams q;
      q.M = M;
      q.N = (int)NJ;
      q.nb1 = E;
      q.nseg = 1;
      q.seg[0].A = Operand{c->Ucat.d() + (side ? (long long)d1 * d1 : 0), M, 1, vstride, 0};
      q.seg[0].B = Operand{side ? EZ : EY, 1, M, J * (side ? L2 : L1), 0};
      q.seg[0].K = M;
      q.tri_upper = 1;
      q.nrm = c->nrmp.d() + (side ? (long long)g1 * E * NJ : 0);
      q.nrm_ld = E * NJ;
      norms.push_back(q);
    }
    nu = c->nrmp.d();
    nw = c->nrmp.d() + (long long)g1 * E * NJ;
    nu_g = nw_g = E * NJ;
    nu_m = nw_m = NJ;
  }

  auto body = [&](int par, cudaStream_t s, cudaGraphConditionalHandle h, int loop) {
    run_gemm(c, rhs_params(Zw), s);
    profiled_other(c, s, [&] {
      modal_uscan(E, nc, d1, J, dt, alpha, c->acoef.d(), c->cden.d(), Rb, Yw, Yw, DYb, EY, cs,
                  s);
    });
    run_gemm(c, g_params(Yw), s);
    profiled_other(c, s, [&] {
      modal_wscan(E, nc, d2, J, c->lam.d(), Rb, Zw, Zw, DZ, EZ,
                  cs, s);
    });
    for (auto& q : norms) run_gemm(c, q, s);
    profiled_other(c, s, [&] {
      modal_decide(E, nc, d1, d2, J, nu, nu_g, nu_m, nw, nw_g, nw_m,
                   (unsigned long long*)c->colmax.p, (unsigned*)c->wticket.p, cs, tol, max_iter,
                   c->rhist.d(), cnt + par, 0, s, h, loop);
    });
    if (!loop)
      PE_CUDA_CHECK(cudaMemcpyAsync(c->pinned_count + par, cnt + par, sizeof(int),
                                    cudaMemcpyDeviceToHost, s));
  };
  const std::vector<const void*> key = {
      (const void*)(intptr_t)4, c->Yb[0].p, c->Zb[0].p, c->R.p, c->DW.p, c->EYZ.p, c->nrmp.p, cs, c->rhist.p, cnt, c->pinned_count, c->RT.p,
      c->GT.p, c->f1t.p, c->cgt.p, c->acoef.p, c->cden.p, c->lam.p, c->Vcat.p, c->Ucat.p, c->colmax.p,
      c->wticket.p,
      (const void*)(intptr_t)max_iter, dkey(alpha), dkey(tol), dkey(dt), LB1, LB2};
  PE_CUDA_CHECK(cudaMemsetAsync(cnt + 2, 0, sizeof(int), st));
  run_sweeps(c, nc, max_iter, key, body, st, true, cnt + 2);

  // final waveforms in the original bases: U = V1 Y, W = V2 Z from each interval's buffer
  basis_gemm(d1, c->Vcat.d(), Yw, d1, (J + 2) * L1, c->Ux_cur.d(), (J + 2) * L1,
             (int)((J + 2) * nc));
  basis_gemm(d2, c->Vcat.d() + (long long)d1 * d1, Zw, d2, (J + 2) * L2, c->Wx_cur.d(),
             (J + 2) * L2, (int)((J + 2) * nc));
  wr_finish(E, nc, d1, d2, J, c->Ux_cur.d(), c->Wx_cur.d(), cs, X_out, sweeps, reasons, st);
  if (resid_hist)
    PE_CUDA_CHECK(cudaMemcpyAsync(resid_hist, c->rhist.p, sizeof(double) * (size_t)E * nc * max_iter,
                                  cudaMemcpyDeviceToDevice, st));
  (void)d;
}

static void fine_allatonce(pe_ctx* c, const double* X_in, double* X_out, int nc, int* sweeps,
                           int* reasons, double* resid_hist, cudaStream_t st,
                           const double* Fload = nullptr) {
  c->wr_last_nc = nc;
  c->wr_last_loads = Fload != nullptr;
  if (Fload) {
    require(c->wr_modal_avail, PE_ERR_ARG,
            "time-dependent loads in the all-at-once solver need symmetric-definite pencils "
            "(A11, M11), (A22, M22) with d1, d2 > 0 (the modal sweep)");
    fine_allatonce_modal(c, X_in, X_out, nc, sweeps, reasons, resid_hist, st, Fload);
    return;
  }
  if (c->wr_modal_full) {
    fine_allatonce_modal(c, X_in, X_out, nc, sweeps, reasons, resid_hist, st);
    return;
  }
  const int d1 = c->d1, d2 = c->d2, E = c->E, J = c->J;
  const long long L1 = (long long)d1 * nc, L2 = (long long)d2 * nc;
  const double alpha = c->wr_alpha, tol = c->wr_tol;
  const int max_iter = c->wr_max_iter;
  c->Ux_cur.ensure(sizeof(double) * E * (J + 2) * L1 + 8);
  c->Ux_new.ensure(sizeof(double) * E * (J + 2) * L1 + 8);
  c->Wx_cur.ensure(sizeof(double) * E * (J + 2) * L2 + 8);
  c->Wx_new.ensure(sizeof(double) * E * (J + 2) * L2 + 8);
  c->R.ensure(sizeof(double) * E * J * L1 + 8);
  const int nk = c->wr_nk;  // half-spectrum modes
  c->P.ensure(sizeof(double) * E * 2 * nk * L1 + 8);
  c->Q.ensure(sizeof(double) * E * 2 * nk * L1 + 8);
  c->DU.ensure(sizeof(double) * E * J * L1 + 8);
  c->DW.ensure(sizeof(double) * E * J * L2 + 8);
  c->V.ensure(sizeof(double) * E * L1 + 8);
  c->colstate.ensure(sizeof(WrColumnState) * E * nc + 8);
  c->nrm.ensure(sizeof(double) * 2 * E * nc * J + 8);
  ensure_zeroed(c->wticket, sizeof(unsigned) * (size_t)E * nc + 8);  // self-resetting tickets
  c->rhist.ensure(sizeof(double) * (size_t)E * nc * max_iter + 8);
  ensure_zeroed(c->splitws, sizeof(double) * (8 * (size_t)E * L1 + 32768));
  c->counter.ensure(sizeof(int) * 2);
  c->stats = FineStats();
  double* Uc = c->Ux_cur.d();
  double* Un = c->Ux_new.d();
  double* Wc = c->Wx_cur.d();
  double* Wn = c->Wx_new.d();
  WrColumnState* cs = (WrColumnState*)c->colstate.p;
  int* cnt = c->counter.i();

  if (c->use_recur && wr_tiny_eligible(d1, d2, J, nk)) {
    // latency regime: the whole WR solve of each interval in one CTA, one launch
    TinyArgsPublic tp{E, d1, d2, J, nk, nc, max_iter, alpha, tol,
                      c->RW.d(), c->M11dt.d(), c->Finv.d(), c->Bk.d(), c->Fw.d(), c->GW.d(),
                      c->cg.d(), c->Emat.d(), c->f1.d(), c->BkT.d(), X_in, X_out, sweeps,
                      reasons, resid_hist, Uc, Wc};
    wr_tiny(tp, st);
    return;
  }
  wr_init(E, nc, d1, d2, J, alpha, X_in, Uc, Un, Wc, Wn, c->V.d(), cs, c->rhist.d(), max_iter, st);
  // W is seeded constant in time, so DW = W_s - W_{s-1} starts at zero; afterwards the
  // commit kernel maintains it for the intervals it commits
  if (d1 && d2) PE_CUDA_CHECK(cudaMemsetAsync(c->DW.p, 0, sizeof(double) * E * J * L2, st));

  // sweep recipe (GEMM parameter blocks are loop-invariant)
  std::vector<GemmParams> pre, post;
  if (d1) {
    GemmParams r;  // R = [-A12 | -M12/dt] [Wx[1..J]; DW] + f1   (build_rhs)
    r.M = d1;
    r.N = J * nc;
    r.nb1 = E;
    r.nseg = d2 ? 2 : 0;
    r.seg[0].A = Operand{c->RW.d(), 2LL * d2, 1, 2LL * d1 * d2, 0};
    r.seg[0].B = Operand{Wc + L2, 1, d2, (J + 2) * L2, 0};
    r.seg[0].K = d2;
    r.seg[1].A = Operand{c->RW.d() + d2, 2LL * d2, 1, 2LL * d1 * d2, 0};
    r.seg[1].B = Operand{c->DW.d(), 1, d2, J * L2, 0};
    r.seg[1].K = d2;
    r.C = c->R.d();
    r.c_i = 1;
    r.c_j = d1;
    r.c_b1 = J * L1;
    r.bias = c->f1.d();
    r.bias_b1 = d1;
    pre.push_back(r);
    GemmParams r0;  // R_0 += M11/dt (u0 - alpha u_final_prev)
    r0.M = d1;
    r0.N = nc;
    r0.nb1 = E;
    r0.nseg = 1;
    r0.seg[0].A = Operand{c->M11dt.d(), d1, 1, (long long)d1 * d1, 0};
    r0.seg[0].B = Operand{c->V.d(), 1, d1, L1, 0};
    r0.seg[0].K = d1;
    r0.C = c->R.d();
    r0.c_i = 1;
    r0.c_j = d1;
    r0.c_b1 = J * L1;
    r0.Cin = c->R.d();
    r0.beta = 1.0;
    r0.ws = c->splitws.d();
    r0.ws_doubles = c->splitws.bytes / sizeof(double);
    pre.push_back(r0);
    GemmParams tf;  // P = S^{-1} R along time (planar re/im per mode, modes 0..nk-1)
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
    pre.push_back(tf);
    GemmParams sh;  // Q_k = (d_k M11 + A11)^{-1} P_k   (einsum, allatonce.py:118)
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
    pre.push_back(sh);
    GemmParams tb;  // U = Re(S Q), conjugate pairs folded into the weights
    tb.M = J;
    tb.N = (int)L1;
    tb.nb1 = E;
    tb.nseg = 1;
    tb.seg[0].A = Operand{c->Fw.d(), 2LL * nk, 1, 0, 0};
    tb.seg[0].B = Operand{c->Q.d(), L1, 1, 2 * nk * L1, 0};
    tb.seg[0].K = 2 * nk;
    tb.C = Un + 2 * L1;
    tb.c_i = L1;
    tb.c_j = 1;
    tb.c_b1 = (J + 2) * L1;
    pre.push_back(tb);
  }
  int rpc_, cs_;
  size_t sm_;
  // modal w recursion (setup_modal): h = V^-1 g by the g GEMM, z scan, W = V Z
  const bool modal = c->wr_modal && c->use_modal && d2 > 0;
  const bool use_rw = !modal && c->use_recur && d2 > 0 && recur_plan(d2, d2, &rpc_, &cs_, &sm_);
  GemmParams gw;  // g_s = [Gu|Gd][U_s; U_{s-1}-U_{s-2}] + dt M22^-T f2   (_w_sweep :222-224)
  GemmParams wb;  // modal back-transform W_s = V Z_s, all s in one launch
  if (d2) {
    gw.M = d2;
    gw.N = J * nc;
    gw.nb1 = E;
    gw.nseg = d1 ? 2 : 0;
    const double* G = modal ? c->GZ.d() : c->GW.d();
    gw.seg[0].A = Operand{G, 2LL * d1, 1, 2LL * d1 * d2, 0};
    gw.seg[0].B = Operand{Un + 2 * L1, 1, d1, (J + 2) * L1, 0};
    gw.seg[0].K = d1;
    gw.seg[1].A = Operand{G + d1, 2LL * d1, 1, 2LL * d1 * d2, 0};
    gw.seg[1].B = Operand{c->DU.d(), 1, d1, J * L1, 0};
    gw.seg[1].K = d1;
    gw.C = Wn + 2 * L2;
    gw.c_i = 1;
    gw.c_j = d2;
    gw.c_b1 = (J + 2) * L2;
    gw.bias = c->cg.d();
    gw.bias_b1 = d2;
    if (modal) {
      c->Z0.ensure(sizeof(double) * E * L2 + 8);
      c->Hz.ensure(sizeof(double) * E * J * L2 + 8);
      gw.C = c->Hz.d();
      gw.c_b1 = J * L2;
      gw.bias = c->cgz.d();
      GemmParams z0;  // Z0 = V^-1 w0, once per solve (w0 is fixed across sweeps)
      z0.M = d2;
      z0.N = nc;
      z0.nb1 = E;
      z0.nseg = 1;
      z0.seg[0].A = Operand{c->Vinv.d(), d2, 1, (long long)d2 * d2, 0};
      z0.seg[0].B = Operand{Wn + L2, 1, d2, (J + 2) * L2, 0};
      z0.seg[0].K = d2;
      z0.C = c->Z0.d();
      z0.c_i = 1;
      z0.c_j = d2;
      z0.c_b1 = L2;
      z0.ws = c->splitws.d();
      z0.ws_doubles = c->splitws.bytes / sizeof(double);
      gemm_f64(z0, st);
      wb.M = d2;
      wb.N = J * nc;
      wb.nb1 = E;
      wb.nseg = 1;
      wb.seg[0].A = Operand{c->Vm.d(), d2, 1, (long long)d2 * d2, 0};
      wb.seg[0].B = Operand{c->Hz.d(), 1, d2, J * L2, 0};
      wb.seg[0].K = d2;
      wb.C = Wn + 2 * L2;
      wb.c_i = 1;
      wb.c_j = d2;
      wb.c_b1 = (J + 2) * L2;
    }
    for (int s = 0; s < J && !use_rw && !modal; ++s) {  // w_{s+1} = E w_s + g_s   (:226-229)
      GemmParams rc;
      rc.M = d2;
      rc.N = nc;
      rc.nb1 = E;
      rc.nseg = 1;
      rc.seg[0].A = Operand{c->Emat.d(), d2, 1, (long long)d2 * d2, 0};
      rc.seg[0].B = Operand{Wn + (s + 1) * L2, 1, d2, (J + 2) * L2, 0};
      rc.seg[0].K = d2;
      rc.C = Wn + (s + 2) * L2;
      rc.c_i = 1;
      rc.c_j = d2;
      rc.c_b1 = (J + 2) * L2;
      rc.Cin = rc.C;
      rc.beta = 1.0;
      // N = nc columns only: split K when the row tiles alone leave SMs idle (cfg3: 64 row
      // tiles x 2 column tiles); the split depends on (M, K, batch) only
      rc.ws = c->splitws.d();
      rc.ws_doubles = c->splitws.bytes / sizeof(double);
      post.push_back(rc);
    }
  }


  // One sweep = ~10 launches (+ J GEMMs when the w recursion does not fit a cluster).
  int* host_cnt = c->pinned_count;
  auto body = [&](int par, cudaStream_t s, cudaGraphConditionalHandle, int) {
    PE_CUDA_CHECK(cudaMemsetAsync(cnt + par, 0, sizeof(int), s));
    for (auto& p : pre) run_gemm(c, p, s);
    if (d1) wr_diff_u(E, nc, d1, J, Un, c->DU.d(), s);
    if (d2) {
      run_gemm(c, gw, s);
      if (modal) {
        wr_modal_scan(E, nc, d2, J, c->lam.d(), c->Z0.d(), c->Hz.d(), s);
        run_gemm(c, wb, s);
      }
      for (auto& p : post) run_gemm(c, p, s);
      if (use_rw)  // all J steps of the w recursion in one cluster-resident launch
        profiled(c, 2.0 * d2 * d2 * nc * E * J, s,
                 [&] { recur_wr(E, d2, nc, J, c->Emat.d(), Wn, s); });
    }
    wr_commit(E, nc, d1, d2, J, alpha, tol, max_iter, 0, Uc, Un, Wc, Wn, c->V.d(), cs,
              c->rhist.d(), cnt + par, c->nrm.d(), (d1 && d2) ? c->DW.d() : nullptr,
              (unsigned*)c->wticket.p, s);
    PE_CUDA_CHECK(cudaMemcpyAsync(host_cnt + par, cnt + par, sizeof(int), cudaMemcpyDeviceToHost, s));
  };
  const std::vector<const void*> key = {
        (const void*)(intptr_t)1,
        Uc, Un, Wc, Wn, c->R.p, c->P.p, c->Q.p, c->DU.p, c->DW.p, c->V.p, cs, c->nrm.p,
        c->rhist.p, cnt, host_cnt, c->splitws.p, c->Bk.p, c->RW.p, c->GW.p, c->Emat.p, c->Finv.p, c->Fw.p,
        c->M11dt.p, c->cg.p, c->f1.p, c->wticket.p, (const void*)(intptr_t)max_iter,
        (const void*)(intptr_t)(c->use_recur ? 1 : 0),
        dkey(alpha), dkey(tol), dkey(c->wr_dt),
        (const void*)(intptr_t)nk, (const void*)(intptr_t)(modal ? 1 : 0), c->Vm.p, c->lam.p,
        c->GZ.p, c->cgz.p, c->Z0.p, c->Hz.p};
  run_sweeps(c, nc, max_iter, key, body, st);
  wr_finish(E, nc, d1, d2, J, Uc, Wc, cs, X_out, sweeps, reasons, st);
  if (resid_hist)
    PE_CUDA_CHECK(cudaMemcpyAsync(resid_hist, c->rhist.p, sizeof(double) * (size_t)E * nc * max_iter,
                                  cudaMemcpyDeviceToDevice, st));
}

// One parareal iteration (parareal.py:188-215): fine sweep on x_0..x_{N-1} of X_old,
// then the fused coarse sweep / correction / norms into X_new.
static void parareal_iterate(pe_ctx* c, int kind, int N, const double* X_old, double* X_new,
                             double* G_cache, double* diff, const int* active, int* wr_sweeps,
                             int* wr_reasons, double* wr_resid, cudaStream_t st) {
  const int E = c->E, d = c->d;
  c->Xin.ensure(sizeof(double) * (size_t)E * N * d + 8);
  c->Xout.ensure(sizeof(double) * (size_t)E * N * d + 8);
  c->partial.ensure(sizeof(double) * (size_t)E * N * 296 * 2 + 8);
  PE_CUDA_CHECK(cudaMemcpy2DAsync(c->Xin.d(), sizeof(double) * N * d, X_old,
                                  sizeof(double) * (N + 1) * d, sizeof(double) * N * d, E,
                                  cudaMemcpyDeviceToDevice, st));
  if (kind == PE_KIND_SEQUENTIAL)  // frozen members: skipped by the ensemble chain kernel
    fine_sequential(c, c->Xin.d(), c->Xout.d(), N, st, nullptr, -1, nullptr, active);
  else
    fine_allatonce(c, c->Xin.d(), c->Xout.d(), N, wr_sweeps, wr_reasons, wr_resid, st);
  if (c->ev_mid) PE_CUDA_CHECK(cudaEventRecord(c->ev_mid, st));
  coarse_correct(E, d, N, c->Phi.d(), c->gG.d(), X_old, c->Xout.d(), G_cache, X_new,
                 c->partial.d(), diff, active, st);
}

}  // namespace pe

using namespace pe;

extern "C" {

const char* pe_last_error(void) { return t_err.c_str(); }
const char* pe_version(void) { return "libpe 0.1 (sm_100a, FP64 DMMA)"; }

int pe_create(pe_ctx** out, int E, int d1, int d2, int max_cols, int J, int device) {
  return guarded([&] {
    require(out != nullptr, PE_ERR_ARG, "ctx out pointer is NULL");
    require(E >= 1 && d1 >= 0 && d2 >= 0 && d1 + d2 >= 1 && max_cols >= 1 && J >= 1,
            PE_ERR_ARG, "need E >= 1, d1, d2 >= 0, d1 + d2 >= 1, max_cols >= 1, J >= 1");
    auto* c = new pe_ctx();
    c->E = E;
    c->d1 = d1;
    c->d2 = d2;
    c->d = d1 + d2;
    c->maxc = max_cols;
    c->J = J;
    c->device = device;
    try {
      bind(c);
      PE_CUDA_CHECK(cudaStreamCreateWithFlags(&c->setup_stream, cudaStreamNonBlocking));
      PE_CUDA_CHECK(cudaStreamCreateWithFlags(&c->work, cudaStreamNonBlocking));
      if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) throw Error{PE_ERR_CUDA, "cublasCreate failed"};
      if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) throw Error{PE_ERR_CUDA, "cusolverDnCreate failed"};
      cublasSetStream(c->blas, c->setup_stream);
      cusolverDnSetStream(c->solver, c->setup_stream);
      PE_CUDA_CHECK(cudaMallocHost(&c->pinned_count, 2 * sizeof(int)));
      const size_t s11 = (size_t)E * d1 * d1, s12 = (size_t)E * d1 * d2, s22 = (size_t)E * d2 * d2;
      c->M11.ensure(8 * s11 + 8);
      c->A11.ensure(8 * s11 + 8);
      c->M12.ensure(8 * s12 + 8);
      c->A12.ensure(8 * s12 + 8);
      c->M22.ensure(8 * s22 + 8);
      c->A22.ensure(8 * s22 + 8);
      c->f1.ensure(8 * (size_t)E * d1 + 8);
      c->f2.ensure(8 * (size_t)E * d2 + 8);
      c->member_set.assign(E, 0);
      c->launches_at_create = g_launches;
    } catch (...) {
      pe_destroy(c);
      throw;
    }
    *out = c;
  });
}

int pe_destroy(pe_ctx* c) {
  if (!c) return PE_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->blas) cublasDestroy(c->blas);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->setup_stream) cudaStreamDestroy(c->setup_stream);
  for (auto& kv : c->sweep_graphs) {
    for (auto ex : kv.second.exec)
      if (ex) cudaGraphExecDestroy(ex);
    if (kv.second.loop) cudaGraphExecDestroy(kv.second.loop);
  }
  if (c->work) cudaStreamDestroy(c->work);
  if (c->pinned_count) cudaFreeHost(c->pinned_count);
  if (c->pinned_diff) cudaFreeHost(c->pinned_diff);
  for (auto e : c->prof_events) cudaEventDestroy(e);
  delete c;
  return PE_OK;
}

int pe_set_system(pe_ctx* c, int m, const double* M11, const double* A11, const double* M12,
                  const double* A12, const double* M22, const double* A22, const double* f1,
                  const double* f2) {
  return guarded([&] {
    require(c != nullptr, PE_ERR_ARG, "ctx is NULL");
    require(m >= 0 && m < c->E, PE_ERR_ARG, "member index out of range");
    bind(c);
    const int d1 = c->d1, d2 = c->d2;
    auto up = [&](DevBuf& b, const double* h, size_t n) {
      if (n == 0) return;
      require(h != nullptr, PE_ERR_ARG, "NULL block for a non-empty subspace");
      PE_CUDA_CHECK(cudaMemcpy(b.d() + (size_t)m * n, h, 8 * n, cudaMemcpyHostToDevice));
    };
    up(c->M11, M11, (size_t)d1 * d1);
    up(c->A11, A11, (size_t)d1 * d1);
    up(c->M12, M12, (size_t)d1 * d2);
    up(c->A12, A12, (size_t)d1 * d2);
    up(c->M22, M22, (size_t)d2 * d2);
    up(c->A22, A22, (size_t)d2 * d2);
    up(c->f1, f1, d1);
    up(c->f2, f2, d2);
    c->member_set[m] = 1;
    c->seq_dt = -1.0;
    c->coarse_dt = -1.0;
    c->wr_ready = false;
  });
}

static void require_system(pe_ctx* c) {
  for (char s : c->member_set) require(s, PE_ERR_STATE, "pe_set_system not called for every member");
}

int pe_prepare_sequential(pe_ctx* c, double dt) {
  return guarded([&] {
    require(c && dt > 0 && std::isfinite(dt), PE_ERR_ARG, "need dt_sub > 0");
    bind(c);
    require_system(c);
    if (c->seq_dt != dt) setup_sequential(c, dt);
  });
}

int pe_prepare_coarse(pe_ctx* c, double dt) {
  return guarded([&] {
    require(c && dt > 0 && std::isfinite(dt), PE_ERR_ARG, "need dt > 0");
    bind(c);
    require_system(c);
    if (c->coarse_dt != dt) setup_coarse(c, dt);
  });
}

int pe_prepare_allatonce(pe_ctx* c, double dt, double alpha, double tol, int max_iter) {
  return guarded([&] {
    require(c && dt > 0, PE_ERR_ARG, "need substeps >= 1 and dt > 0");
    require(alpha > 0.0 && alpha < 1.0, PE_ERR_ARG, "alpha must lie in (0, 1)");
    require(max_iter >= 1, PE_ERR_ARG, "max_iter must be >= 1");
    bind(c);
    require_system(c);
    if (!(c->wr_ready && c->wr_dt == dt && c->wr_alpha == alpha)) setup_allatonce(c, dt, alpha, tol, max_iter);
    c->wr_tol = tol;
    c->wr_max_iter = max_iter;
  });
}

int pe_fine_sequential(pe_ctx* c, const double* X_in, double* X_out, int nc, void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && nc >= 1 && nc <= c->maxc, PE_ERR_ARG, "bad fine_sequential arguments");
    require(c->seq_dt > 0, PE_ERR_STATE, "pe_prepare_sequential not called");
    bind(c);
    fine_sequential(c, X_in, X_out, nc, (cudaStream_t)stream);
  });
}

int pe_fine_allatonce(pe_ctx* c, const double* X_in, double* X_out, int nc, int* sweeps,
                      int* reasons, double* resid_hist, void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && nc >= 1 && nc <= c->maxc, PE_ERR_ARG, "bad fine_allatonce arguments");
    require(c->wr_ready, PE_ERR_STATE, "pe_prepare_allatonce not called");
    bind(c);
    fine_allatonce(c, X_in, X_out, nc, sweeps, reasons, resid_hist, (cudaStream_t)stream);
  });
}

int pe_coarse_correct(pe_ctx* c, int N, const double* X_old, const double* F_hat,
                      double* G_cache, double* X_new, double* diff, const int* active,
                      void* stream) {
  return guarded([&] {
    require(c && X_old && X_new && G_cache && N >= 1, PE_ERR_ARG, "bad coarse_correct arguments");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    bind(c);
    c->partial.ensure(sizeof(double) * (size_t)c->E * N * 296 * 2 + 8);
    coarse_correct(c->E, c->d, N, c->Phi.d(), c->gG.d(), X_old, F_hat, G_cache, X_new,
                   c->partial.d(), diff, active, (cudaStream_t)stream);
  });
}

int pe_fine_sequential_loads(pe_ctx* c, const double* X_in, double* X_out, int nc,
                             const double* F, void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && F && nc >= 1, PE_ERR_ARG, "bad fine_sequential_loads arguments");
    require(c->seq_dt > 0, PE_ERR_STATE, "pe_prepare_sequential not called");
    bind(c);
    fine_sequential(c, X_in, X_out, nc, (cudaStream_t)stream, nullptr, -1, F);
  });
}

int pe_split_step_loads(pe_ctx* c, const double* X_in, const double* X_prev, double* X_out,
                        int nc, const double* F, void* stream) {
  return guarded([&] {
    require(c && X_in && X_prev && X_out && F && nc >= 1, PE_ERR_ARG, "bad split_step_loads arguments");
    require(c->seq_dt > 0, PE_ERR_STATE, "pe_prepare_sequential not called");
    bind(c);
    fine_sequential(c, X_in, X_out, nc, (cudaStream_t)stream, X_prev, 1, F);
  });
}

int pe_fine_allatonce_loads(pe_ctx* c, const double* X_in, double* X_out, int nc,
                            const double* F, int* sweeps, int* reasons, double* resid_hist,
                            void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && F && nc >= 1 && nc <= c->maxc, PE_ERR_ARG,
            "bad fine_allatonce_loads arguments");
    require(c->wr_ready, PE_ERR_STATE, "pe_prepare_allatonce not called");
    bind(c);
    fine_allatonce(c, X_in, X_out, nc, sweeps, reasons, resid_hist, (cudaStream_t)stream, F);
  });
}

int pe_coarse_correct_loads(pe_ctx* c, int N, const double* X_old, const double* F_hat,
                            double* G_cache, double* X_new, double* diff, const int* active,
                            const double* Fc, void* stream) {
  return guarded([&] {
    require(c && X_old && X_new && G_cache && Fc && N >= 1, PE_ERR_ARG,
            "bad coarse_correct_loads arguments");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    bind(c);
    cudaStream_t st = (cudaStream_t)stream;
    c->partial.ensure(sizeof(double) * (size_t)c->E * N * 296 * 2 + 8);
    const double* gs = coarse_load_terms(c, N, Fc, st);
    coarse_correct(c->E, c->d, N, c->Phi.d(), c->gG.d(), X_old, F_hat, G_cache, X_new,
                   c->partial.d(), diff, active, st, gs);
  });
}

int pe_coarse_apply_loads(pe_ctx* c, const double* X_in, double* X_out, int nc,
                          const double* Fc, void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && Fc && nc >= 1, PE_ERR_ARG, "bad coarse_apply_loads arguments");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    bind(c);
    cudaStream_t st = (cudaStream_t)stream;
    const int d = c->d, E = c->E;
    c->hist_tmp.ensure(sizeof(double) * (size_t)E * 2 * d + 8);
    c->Gc.ensure(sizeof(double) * (size_t)E * d + 8);
    c->partial.ensure(sizeof(double) * (size_t)E * 296 * 2 + 8);
    const double* gs = coarse_load_terms(c, nc, Fc, st);  // (E, nc, d): one term per state
    c->Xs.ensure(sizeof(double) * (size_t)E * d + 8);
    for (int n = 0; n < nc; ++n) {
      PE_CUDA_CHECK(cudaMemcpy2DAsync(c->hist_tmp.d(), sizeof(double) * 2 * d, X_in + (size_t)n * d,
                                      sizeof(double) * nc * d, sizeof(double) * d, E,
                                      cudaMemcpyDeviceToDevice, st));
      PE_CUDA_CHECK(cudaMemcpy2DAsync(c->Xs.d(), sizeof(double) * d, gs + (size_t)n * d,
                                      sizeof(double) * nc * d, sizeof(double) * d, E,
                                      cudaMemcpyDeviceToDevice, st));
      coarse_correct(E, d, 1, c->Phi.d(), c->gG.d(), c->hist_tmp.d(), nullptr, c->Gc.d(),
                     c->hist_tmp.d(), c->partial.d(), nullptr, nullptr, st, c->Xs.d());
      PE_CUDA_CHECK(cudaMemcpy2DAsync(X_out + (size_t)n * d, sizeof(double) * nc * d,
                                      c->hist_tmp.d() + d, sizeof(double) * 2 * d,
                                      sizeof(double) * d, E, cudaMemcpyDeviceToDevice, st));
    }
  });
}

int pe_coarse_apply(pe_ctx* c, const double* X_in, double* X_out, int nc, void* stream) {
  return guarded([&] {
    require(c && X_in && X_out && nc >= 1, PE_ERR_ARG, "bad coarse_apply arguments");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    bind(c);
    cudaStream_t st = (cudaStream_t)stream;
    const int d = c->d, E = c->E;
    c->hist_tmp.ensure(sizeof(double) * (size_t)E * 2 * d + 8);
    c->Gc.ensure(sizeof(double) * (size_t)E * d + 8);
    c->partial.ensure(sizeof(double) * (size_t)E * 296 * 2 + 8);
    for (int n = 0; n < nc; ++n) {
      // one-interval initial sweep: row 1 = G(row 0), same kernel as the fused sweep
      PE_CUDA_CHECK(cudaMemcpy2DAsync(c->hist_tmp.d(), sizeof(double) * 2 * d, X_in + (size_t)n * d,
                                      sizeof(double) * nc * d, sizeof(double) * d, E,
                                      cudaMemcpyDeviceToDevice, st));
      coarse_correct(E, d, 1, c->Phi.d(), c->gG.d(), c->hist_tmp.d(), nullptr, c->Gc.d(),
                     c->hist_tmp.d(), c->partial.d(), nullptr, nullptr, st);
      PE_CUDA_CHECK(cudaMemcpy2DAsync(X_out + (size_t)n * d, sizeof(double) * nc * d,
                                      c->hist_tmp.d() + d, sizeof(double) * 2 * d,
                                      sizeof(double) * d, E, cudaMemcpyDeviceToDevice, st));
    }
  });
}

int pe_parareal_run(pe_ctx* c, int kind, int N, const double* X0, int k_max, double epsilon,
                    int rule, double* history, double* diffs_h, int* iters_h, int* conv_h,
                    int* wr_sweeps, int* wr_reasons, double* wr_resid, float* fine_ms_h,
                    float* coarse_ms_h, int* k_done, void* stream) {
  return guarded([&] {
    require(c && X0 && history && N >= 1 && N <= c->maxc && k_max >= 0, PE_ERR_ARG,
            "bad parareal_run arguments");
    require(kind == PE_KIND_SEQUENTIAL || kind == PE_KIND_ALLATONCE, PE_ERR_ARG,
            "unknown fine propagator kind");
    require(rule == PE_RULE_ABSOLUTE || rule == PE_RULE_RELATIVE, PE_ERR_ARG, "unknown stop rule");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    require(kind == PE_KIND_SEQUENTIAL ? c->seq_dt > 0 : c->wr_ready, PE_ERR_STATE,
            "fine propagator not prepared");
    bind(c);
    cudaStream_t st = (cudaStream_t)stream;
    const int E = c->E, d = c->d;
    const size_t slab = (size_t)E * (N + 1) * d;
    auto H = [&](int k) { return history + (size_t)k * slab; };
    c->Gc.ensure(sizeof(double) * (size_t)E * N * d + 8);
    c->partial.ensure(sizeof(double) * (size_t)E * N * 296 * 2 + 8);
    c->diff.ensure(sizeof(double) * 2 * E + 8);
    c->active.ensure(sizeof(int) * E + 8);
    if (c->pinned_diff_n < (size_t)2 * E) {
      if (c->pinned_diff) cudaFreeHost(c->pinned_diff);
      PE_CUDA_CHECK(cudaMallocHost(&c->pinned_diff, sizeof(double) * 2 * E));
      c->pinned_diff_n = 2 * E;
    }
    std::vector<int> act(E, 1);
    for (int e = 0; e < E; ++e) {
      iters_h[e] = 0;
      conv_h[e] = 0;
    }
    PE_CUDA_CHECK(cudaMemcpyAsync(c->active.p, act.data(), sizeof(int) * E, cudaMemcpyHostToDevice, st));
    // x_0 into row 0 of every member, then the initial coarse sweep (parareal.py:150-157)
    PE_CUDA_CHECK(cudaMemcpy2DAsync(H(0), sizeof(double) * (N + 1) * d, X0, sizeof(double) * d,
                                    sizeof(double) * d, E, cudaMemcpyDeviceToDevice, st));
    coarse_correct(E, d, N, c->Phi.d(), c->gG.d(), H(0), nullptr, c->Gc.d(), H(0),
                   c->partial.d(), nullptr, nullptr, st);
    cudaEvent_t e0, e1, e2;
    PE_CUDA_CHECK(cudaEventCreate(&e0));
    PE_CUDA_CHECK(cudaEventCreate(&e1));
    PE_CUDA_CHECK(cudaEventCreate(&e2));
    int k = 0;
    int n_active = E;
    for (k = 1; k <= k_max && n_active > 0; ++k) {
      PE_CUDA_CHECK(cudaEventRecord(e0, st));
      const size_t off = (size_t)(k - 1) * E * N;
      c->ev_mid = e1;
      parareal_iterate(c, kind, N, H(k - 1), H(k), c->Gc.d(), c->diff.d(), c->active.i(),
                       wr_sweeps ? wr_sweeps + off : nullptr,
                       wr_reasons ? wr_reasons + off : nullptr,
                       wr_resid ? wr_resid + off * c->wr_max_iter : nullptr, st);
      c->ev_mid = nullptr;
      PE_CUDA_CHECK(cudaEventRecord(e2, st));
      PE_CUDA_CHECK(cudaMemcpyAsync(c->pinned_diff, c->diff.p, sizeof(double) * 2 * E,
                                    cudaMemcpyDeviceToHost, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
      float fm = 0, cm = 0;
      PE_CUDA_CHECK(cudaEventElapsedTime(&fm, e0, e1));
      PE_CUDA_CHECK(cudaEventElapsedTime(&cm, e1, e2));
      if (fine_ms_h) fine_ms_h[k - 1] = fm;
      if (coarse_ms_h) coarse_ms_h[k - 1] = cm;
      bool changed = false;
      for (int e = 0; e < E; ++e) {
        double v = NAN;
        if (act[e]) {
          const double num = c->pinned_diff[2 * e], den = c->pinned_diff[2 * e + 1];
          v = (rule == PE_RULE_ABSOLUTE) ? num : (den > 0 ? num / den : num);
          iters_h[e] = k;
          if (v < epsilon) {
            conv_h[e] = 1;
            act[e] = 0;
            --n_active;
            changed = true;
          }
        }
        if (diffs_h) diffs_h[(size_t)(k - 1) * E + e] = v;
      }
      if (changed && n_active > 0)
        PE_CUDA_CHECK(cudaMemcpyAsync(c->active.p, act.data(), sizeof(int) * E, cudaMemcpyHostToDevice, st));
      PE_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    if (k_done) *k_done = k - 1;
  });
}

int pe_split_step(pe_ctx* c, const double* X_in, const double* X_prev, double* X_out, int nc,
                  void* stream) {
  return guarded([&] {
    require(c && X_in && X_prev && X_out && nc >= 1, PE_ERR_ARG, "bad split_step arguments");
    require(c->seq_dt > 0, PE_ERR_STATE, "pe_prepare_sequential not called");
    bind(c);
    fine_sequential(c, X_in, X_out, nc, (cudaStream_t)stream, X_prev, 1);
  });
}

int pe_wr_waveforms(pe_ctx* c, double* U_out, double* W_out, int nc, void* stream) {
  return guarded([&] {
    require(c && nc >= 1, PE_ERR_ARG, "bad wr_waveforms arguments");
    require(c->wr_ready && c->Ux_cur.p, PE_ERR_STATE, "no all-at-once solve to read back");
    bind(c);
    cudaStream_t st = (cudaStream_t)stream;
    if (U_out && c->d1) wr_gather(c->E, nc, c->d1, c->J, c->Ux_cur.d(), U_out, st);
    if (W_out && c->d2) wr_gather(c->E, nc, c->d2, c->J, c->Wx_cur.d(), W_out, st);
  });
}

int pe_parareal_iterate(pe_ctx* c, int kind, int N, const double* X_old, double* X_new,
                        double* G_cache, double* diff, const int* active, int* wr_sweeps,
                        int* wr_reasons, double* wr_resid, void* stream) {
  return guarded([&] {
    require(c && X_old && X_new && G_cache && N >= 1 && N <= c->maxc, PE_ERR_ARG,
            "bad parareal_iterate arguments");
    require(kind == PE_KIND_SEQUENTIAL || kind == PE_KIND_ALLATONCE, PE_ERR_ARG,
            "unknown fine propagator kind");
    require(c->coarse_dt > 0, PE_ERR_STATE, "pe_prepare_coarse not called");
    require(kind == PE_KIND_SEQUENTIAL ? c->seq_dt > 0 : c->wr_ready, PE_ERR_STATE,
            "fine propagator not prepared");
    bind(c);
    parareal_iterate(c, kind, N, X_old, X_new, G_cache, diff, active, wr_sweeps, wr_reasons,
                     wr_resid, (cudaStream_t)stream);
  });
}

int pe_set_recurrence(pe_ctx* c, int on) {
  return guarded([&] {
    require(c != nullptr, PE_ERR_ARG, "ctx is NULL");
    c->use_recur = on != 0;
  });
}

int pe_set_modal(pe_ctx* c, int on) {
  return guarded([&] {
    require(c != nullptr, PE_ERR_ARG, "ctx is NULL");
    if (c->use_modal != (on != 0)) c->wr_ready = false;  // operators depend on the choice
    c->use_modal = on != 0;
  });
}

int pe_wr_is_modal(pe_ctx* c) {
  if (!c) return PE_ERR_ARG;
  if (!c->wr_ready) return 0;
  return c->wr_modal_full ? 2 : (c->wr_modal ? 1 : 0);
}

int pe_set_profiling(pe_ctx* c, int on) {
  return guarded([&] {
    require(c != nullptr, PE_ERR_ARG, "ctx is NULL");
    c->profiling = on != 0;
    c->prof_used = 0;
  });
}

int pe_gemm_f64(int M, int N, int K, int batch, const double* A, long long a_i, long long a_k,
                long long a_b, const double* B, long long b_k, long long b_j, long long b_b,
                double* C, long long c_i, long long c_j, long long c_b, void* stream) {
  return guarded([&] {
    require(M >= 0 && N >= 0 && K >= 0 && batch >= 1 && C, PE_ERR_ARG, "bad gemm arguments");
    GemmParams p;
    p.M = M;
    p.N = N;
    p.nb1 = batch;
    p.nseg = K > 0 ? 1 : 0;
    p.seg[0].A = Operand{A, a_i, a_k, a_b, 0};
    p.seg[0].B = Operand{B, b_k, b_j, b_b, 0};
    p.seg[0].K = K;
    p.C = C;
    p.c_i = c_i;
    p.c_j = c_j;
    p.c_b1 = c_b;
    gemm_f64(p, (cudaStream_t)stream);
  });
}

int pe_batched_inverse(int n, int batch, const double* A, double* Ainv, int* info,
                       void* stream) {
  return guarded([&] {
    require(n >= 1 && batch >= 1 && A && Ainv, PE_ERR_ARG, "bad batched-inverse arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t tot = (size_t)batch * n * n;
    DevBuf lu, piv, dinfo;
    lu.ensure(sizeof(double) * tot);
    piv.ensure(sizeof(int) * (size_t)batch * n);
    dinfo.ensure(sizeof(int) * (size_t)batch);
    PE_CUDA_CHECK(cudaMemcpyAsync(lu.p, A, sizeof(double) * tot, cudaMemcpyDeviceToDevice, st));
    batched_lu_inverse(n, batch, lu.d(), Ainv, piv.i(), dinfo.i(), st);
    std::vector<int> h((size_t)batch);
    PE_CUDA_CHECK(cudaMemcpyAsync(h.data(), dinfo.p, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
    PE_CUDA_CHECK(cudaStreamSynchronize(st));
    if (info) std::copy(h.begin(), h.end(), info);
  });
}

int pe_shifted_inverses(int d1, int J, double dt, double alpha, const double* M11,
                        const double* A11, double* inv_re, double* inv_im, void* stream) {
  return guarded([&] {
    require(d1 >= 1 && J >= 1 && dt > 0 && alpha > 0 && M11 && A11 && inv_re && inv_im,
            PE_ERR_ARG, "bad shifted-inverse arguments");
    shifted_inverses(d1, J, dt, alpha, M11, A11, inv_re, inv_im, (cudaStream_t)stream);
  });
}

long long pe_launch_count(pe_ctx* c) { return c ? g_launches - c->launches_at_create : g_launches; }

int pe_last_fine_other_ms(pe_ctx* c, double* other_ms) {
  return guarded([&] {
    require(c != nullptr && other_ms != nullptr, PE_ERR_ARG, "bad arguments");
    *other_ms = c->stats.other_ms;
  });
}

int pe_last_fine_stats(pe_ctx* c, double* gemm_ms, double* gemm_flops_out, int* launches) {
  return guarded([&] {
    require(c != nullptr, PE_ERR_ARG, "ctx is NULL");
    if (gemm_ms) *gemm_ms = c->stats.gemm_ms;
    if (gemm_flops_out) *gemm_flops_out = c->stats.gemm_flops;
    if (launches) *launches = c->stats.launches;
  });
}

}  // extern "C"
