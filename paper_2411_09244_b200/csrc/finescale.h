// Shared between the fine reference solvers (finescale.cu: dense K^-1 paths; finechain.cu:
// block-tridiagonal chain solver for large grids).
#pragma once

#include <cuda_runtime.h>

namespace pe {

struct RefSolveArgs {
  int n;
  const int *mp, *mi, *ap, *ai;
  const double *mv, *av, *b, *u0;
  double t_end;
  int n_steps;
  double* states_h;
  int keep;
  cudaStream_t st;
  float* step_ms;
};

// v(i) = (M u)(i) / dt + b(i), i < n (device CSR of M)
void fine_rhs(int n, const int* mp, const int* mi, const double* mv, double inv_dt,
              const double* u, const double* b, double* v, cudaStream_t st);

// Banded operator, large enough (or PE_FINE_CHAIN=1): the chain solver applies
bool fine_chain_applicable(int n, const int* mp, const int* mi, const int* ap, const int* ai,
                           int* block = nullptr);
void fine_chain_solve(RefSolveArgs& a);

}  // namespace pe
