// Internal declarations shared by the libpe translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

namespace pe {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};

#define PE_CUDA_CHECK(expr)                                                               \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::pe::Error{PE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

// ---------------------------------------------------------------- launches
// Programmatic dependent launch (PDL): the sweep kernels are launched with programmatic
// stream serialization, so a kernel's CTAs are scheduled while its predecessor drains.
// Every such kernel first triggers its own dependents (all of its CTAs are resident by
// then) and then waits for its predecessor grid to complete and flush before touching any
// global memory; because every kernel of the chain waits, completion stays transitive.
extern bool g_pdl;
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = g_pdl ? at : nullptr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  PE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ---------------------------------------------------------------- FP64 DMMA GEMM
//
// C[z](i,j) = alpha * sum_seg sum_k A_seg[z](i,k) B_seg[z](k,j)
//             + beta * Cin[z](i,j) + bias[z](i)            (then optional D = C - Xp)
// with z = z1 * nb2 + z2 a two-level batch index; every operand has arbitrary
// element strides and per-level batch strides (0 = shared across that level).
// The k reduction runs segment by segment, k ascending, in m8n8k4 DMMA steps, so
// the result for one (i,j) does not depend on tile shape or on the other columns
// (batch invariance: F applied to one state equals F applied inside a batch).
struct Operand {
  const double* p = nullptr;
  long long s0 = 0, s1 = 0;    // element strides (A: i,k  B: k,j)
  long long b1 = 0, b2 = 0;    // batch strides (level 1, level 2)
};

struct GemmSeg {
  Operand A, B;
  int K = 0;
};

struct GemmParams {
  int M = 0, N = 0;
  int nb1 = 1, nb2 = 1;
  int nseg = 0;
  GemmSeg seg[3];
  double* C = nullptr;
  long long c_i = 0, c_j = 0, c_b1 = 0, c_b2 = 0;
  double alpha = 1.0;
  double beta = 0.0;
  const double* Cin = nullptr;  // same strides as C
  const double* bias = nullptr;
  long long bias_b1 = 0, bias_b2 = 0;
  // norm epilogue (no C output): for every 8-row block g of C and column j of batch z,
  // nrm[g * nrm_ld + z * N + j] = sum of the block's squared entries, summed in a fixed
  // xor-shuffle order that does not depend on the tile shape (batch invariance)
  double* nrm = nullptr;
  long long nrm_ld = 0;
  // A (single segment) is upper triangular: k-tiles entirely left of a row tile's first
  // row hold exact zeros and are skipped (their DMMA steps would add +0)
  int tri_upper = 0;
  double* D = nullptr;          // optional D = C - Xp, same strides as C
  const double* Xp = nullptr;
  // split-K for skinny launches: partial tiles go to `ws`, a reduction kernel sums the
  // splits in order and applies the epilogue.  The split factor depends only on
  // (M, K, batch), never on N (batch invariance).  ws == nullptr disables splitting.
  double* ws = nullptr;
  size_t ws_doubles = 0;
  int ksplit = 1;  // set by gemm_f64
  int raster = 0;  // set by gemm_f64: grouped tile rasterisation (row tiles per group)
};

// Launch; chooses tile shape and the k-/j-contiguous loader variant from strides.
void gemm_f64(const GemmParams& p, cudaStream_t st);
// Row-balanced persistent launch for batched skinny products (ensemble fine step); rows
// below zero_rows have exact zeros in the second segment's k-range [zero_k0, zero_k1)
// (segment-local), skipped.  Only for shapes with gemm_rowbalanced_eligible(p).
bool gemm_rowbalanced_eligible(const GemmParams& p, int zero_rows, int zero_k0, int zero_k1);
void gemm_f64_rowbalanced(const GemmParams& p, int zero_rows, int zero_k0, int zero_k1,
                          cudaStream_t st);
// J chained steps X_{s+1} = T [X_s ; D_s] + c in one cooperative launch (p2: the two-segment
// step's parameters; D_in may be null: the first step then has one segment).  bufX / bufD
// are ping-pong state buffers, cnt holds nb1 counters.  active (nb1 ints, device) or null:
// members with 0 are skipped (their X_out rows are not written).
bool gemm_rowbalanced_chain_eligible(const GemmParams& p2, int zero_rows, int zero_k0, int zero_k1);
void gemm_f64_rowbalanced_chain(const GemmParams& p2, int zero_rows, int zero_k0, int zero_k1, int J,
                                const double* X_in, const double* D_in, double* const bufX[2],
                                double* const bufD[2], double* X_out, unsigned* cnt,
                                const int* active, cudaStream_t st);
// Flop count of one launch (2*M*N*sumK*batch), for the roofline bookkeeping.
double gemm_flops(const GemmParams& p);

// ---------------------------------------------------------------- batched inversion (batchlu.cu)
// Ainv[b] = A[b]^-1 for `batch` row-major n x n matrices (batch stride n*n).  A is
// overwritten by its LU factors; piv: batch*n ints; info: batch ints (device), 0 or the
// 1-based index of the first zero pivot.  Enqueued on st, no host synchronisation.
void batched_lu_inverse(int n, int batch, double* A, double* Ainv, int* piv, int* info,
                        cudaStream_t st);
// inv(d_k M11 + A11) for every time mode, planar (J, d1, d1) outputs (allatonce.py:100-110)
void shifted_inverses(int d1, int J, double dt, double alpha, const double* M11,
                      const double* A11, double* inv_re, double* inv_im, cudaStream_t st);

// ---------------------------------------------------------------- WR helpers
struct WrColumnState {
  int active;
  int iterations;
  int stall;
  int reason;
  double prev;
  double r0;
  int fpar;  // reserved (buffer index of the interval's latest waveforms; 0 in place)
  int pad;
};

void wr_init(int E, int ncols, int d1, int d2, int J, double alpha, const double* X_in,
             double* Ux_cur, double* Ux_new, double* Wx_cur, double* Wx_new, double* V,
             WrColumnState* cs, double* resid_hist, int max_iter, cudaStream_t st);
void wr_diff_u(int E, int ncols, int d1, int J, const double* Ux_new, double* DU,
               cudaStream_t st);
void wr_commit(int E, int ncols, int d1, int d2, int J, double alpha, double tol,
               int max_iter, int sweep, double* Ux_cur, const double* Ux_new, double* Wx_cur,
               const double* Wx_new, double* V, WrColumnState* cs, double* resid_hist,
               int* active_count, double* nrm, double* DW, unsigned* ticket, cudaStream_t st);
void wr_finish(int E, int ncols, int d1, int d2, int J, const double* Ux_cur,
               const double* Wx_cur, const WrColumnState* cs, double* X_out, int* sweeps,
               int* reasons, cudaStream_t st);

void wr_modal_scan(int E, int nc, int d2, int J, const double* lam, const double* Z0, double* Z,
                   cudaStream_t st);
void wr_gather(int E, int nc, int dd, int J, const double* X, double* out, cudaStream_t st);

// ---------------------------------------------------------------- modal WR (wr_modal.cu)
void wr_state_init(long long ncs, WrColumnState* cs, double* resid_hist, int max_iter,
                   cudaStream_t st);
void modal_seed(int E, int nc, int d1, int d2, int J, const double* Y0, const double* Z0,
                double* Yb0, double* Yb1, double* Zb0, double* Zb1, double* DZ, cudaStream_t st);
void modal_uscan(int E, int nc, int d1, int J, double dt, double alpha, const double* acoef,
                 const double* cden, const double* R, const double* Yc, double* Yn, double* DY,
                 double* EY, const WrColumnState* cs, cudaStream_t st);
void modal_wscan(int E, int nc, int d2, int J, const double* lam, const double* H,
                 const double* Zc, double* Zn, double* DZ, double* EZ, const WrColumnState* cs,
                 cudaStream_t st);
void modal_decide(int E, int nc, int d1, int d2, int J, const double* nu, long long nu_g,
                  long long nu_m, const double* nw, long long nw_g, long long nw_m,
                  unsigned long long* colmax, unsigned* ticket, WrColumnState* cs, double tol,
                  int max_iter, double* resid_hist, int* active_count, int par_new,
                  cudaStream_t st, cudaGraphConditionalHandle cond = 0, int use_cond = 0);

void sub(long long n, const double* a, const double* b, double* out, cudaStream_t st);

// ---------------------------------------------------------------- recurrences (recur.cu)
bool recur_plan(int M, int KT, int* rpc, int* cs, size_t* smem, int nclusters = 0);
// sequential fine chain on all SMs when T is too large for one cluster (seqgrid.cu)
bool seqgrid_fits(int E, int d1, int d2, int nc);
bool seqgrid_seq(int d1, int d2, int nc, int S, const double* T, const double* c,
                 const double* Xin, double* Xout, double* Z, unsigned* cnt, cudaStream_t st);
bool recur_wr(int E, int d2, int nc, int J, const double* Emat, double* Wx, cudaStream_t st);
bool recur_seq(int E, int d, int nc, int S, const double* T, const double* c, const double* Xin,
               double* Xout, double* scratch, cudaStream_t st);

// ---------------------------------------------------------------- fused small-problem WR
struct TinyArgsPublic {
  int E, d1, d2, J, npm, nc, max_iter;
  double alpha, tol;
  const double *RW, *M11dt, *Finv, *Bk, *Fw, *GW, *cg, *Emat, *f1;
  const double* BkT;
  const double* X_in;
  double* X_out;
  int* sweeps;
  int* reasons;
  double* resid_hist;
  double *Ux_cur, *Wx_cur;
};
bool wr_tiny_eligible(int d1, int d2, int J, int npm);
void transpose_blocks(int nblocks, int n, const double* src, double* dst, cudaStream_t st);
void wr_tiny(const TinyArgsPublic& p, cudaStream_t st);

// ---------------------------------------------------------------- coarse sweep
// Row-partitioned cluster kernel; see coarse.cu.
void coarse_correct(int E, int d, int N, const double* Phi, const double* gvec,
                    const double* X_old, const double* F_hat, double* G_cache, double* X_new,
                    double* partial, double* diff, const int* active, cudaStream_t st, const double* gseries = nullptr);
int coarse_cluster_size(int d);

extern long long g_launches;  // kernel launches issued by libpe in this process

}  // namespace pe
