// Timing probe for the ensemble coarse stream (cfg4 shape: E = 64, d = 600, N = 32):
// links one version of coarse.cu and times coarse_correct with CUDA events.
//   nvcc ... coarse_stream_probe.cu <coarse.cu variant> -o probe [-DOLD]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

namespace pe {
long long g_launches = 0;
#ifdef OLD
void coarse_correct(int E, int d, int N, const double* Phi, const double* gvec,
                    const double* X_old, const double* F_hat, double* G_cache, double* X_new,
                    double* partial, double* diff, const int* active, cudaStream_t st);
#else
void coarse_correct(int E, int d, int N, const double* Phi, const double* gvec,
                    const double* X_old, const double* F_hat, double* G_cache, double* X_new,
                    double* partial, double* diff, const int* active, cudaStream_t st,
                    const double* gseries);
#endif
}  // namespace pe

int main(int argc, char** argv) {
  const int E = argc > 1 ? atoi(argv[1]) : 64, d = argc > 2 ? atoi(argv[2]) : 600,
            N = argc > 3 ? atoi(argv[3]) : 32;
  const size_t nphi = (size_t)E * d * d;
  std::vector<double> h(nphi);
  for (size_t i = 0; i < nphi; ++i) h[i] = ((double)((i * 2654435761u) % 1000) - 500.0) * 1e-6;
  double *Phi, *g, *Xo, *Fh, *Gc, *Xn, *part, *diff;
  cudaMalloc(&Phi, nphi * 8);
  cudaMemcpy(Phi, h.data(), nphi * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&g, (size_t)E * d * 8);
  cudaMalloc(&Xo, (size_t)E * (N + 1) * d * 8);
  cudaMalloc(&Xn, (size_t)E * (N + 1) * d * 8);
  cudaMalloc(&Fh, (size_t)E * N * d * 8);
  cudaMalloc(&Gc, (size_t)E * N * d * 8);
  cudaMalloc(&part, (size_t)E * N * 600 * 2 * 8);
  cudaMalloc(&diff, (size_t)E * 2 * 8);
  cudaMemset(g, 0, (size_t)E * d * 8);
  cudaMemset(Xo, 0, (size_t)E * (N + 1) * d * 8);
  cudaMemset(Fh, 0, (size_t)E * N * d * 8);
  cudaMemset(Gc, 0, (size_t)E * N * d * 8);
  auto run = [&] {
#ifdef OLD
    pe::coarse_correct(E, d, N, Phi, g, Xo, Fh, Gc, Xn, part, diff, nullptr, 0);
#else
    pe::coarse_correct(E, d, N, Phi, g, Xo, Fh, Gc, Xn, part, diff, nullptr, 0, nullptr);
#endif
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 10;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / reps / N;
  printf("E=%d d=%d N=%d: %.2f us per coarse step, %.0f GB/s of Phi  (%s)\n", E, d, N, us,
         nphi * 8.0 / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
