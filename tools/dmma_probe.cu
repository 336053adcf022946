// DMMA m8n8k4 f64 latency / throughput and DFMA throughput on B200.
#include <cstdio>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void k_dmma(int iters, double* out, long long* cyc) {
  double c[CHAINS][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CHAINS>
__global__ void k_dfma(int iters, double* out) {
  double c[CHAINS];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps issue DMMA chains, the other half DFMA chains: do the two share a pipe?
__global__ void k_mixed(int iters, int dfma_iters, double* out) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if ((warp >> 2) & 1) {  // warps 4-7: DFMA on all four SMSPs; warps 0-3: DMMA
    double c[8];
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
  } else {
    double c[8][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  auto run_dmma = [&](auto kern, int chains, int blocks, int threads) {
    kern<<<blocks, threads>>>(100, out, cyc);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(iters, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double flops = 512.0 * chains * iters * (double)blocks * (threads / 32);
    printf("DMMA chains=%d blocks=%d warps/blk=%d: %.2f cyc per dependent DMMA-step, %.2f TFLOP/s\n",
           chains, blocks, threads / 32, (double)c / iters, flops / ms / 1e9);
  };
  run_dmma(k_dmma<1>, 1, 1, 32);
  run_dmma(k_dmma<4>, 4, 1, 32);
  run_dmma(k_dmma<8>, 8, 1, 32);
  run_dmma(k_dmma<1>, 1, 148, 128);
  run_dmma(k_dmma<4>, 4, 148, 128);
  run_dmma(k_dmma<4>, 4, 148, 256);
  run_dmma(k_dmma<8>, 8, 148, 256);
  run_dmma(k_dmma<8>, 8, 296, 256);
  auto run_dfma = [&](auto kern, int chains, int blocks, int threads) {
    kern<<<blocks, threads>>>(100, out);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * chains * iters * (double)blocks * threads;
    printf("DFMA chains=%d blocks=%d threads=%d: %.2f TFLOP/s\n", chains, blocks, threads,
           flops / ms / 1e9);
  };
  run_dfma(k_dfma<4>, 4, 148, 256);
  run_dfma(k_dfma<8>, 8, 296, 256);
  run_dfma(k_dfma<8>, 8, 592, 256);
  for (int dfi : {0, 8000, 16000, 32000, 64000}) {
    k_mixed<<<148, 256>>>(100, 100, out);
    cudaEventRecord(a);
    k_mixed<<<148, 256>>>(iters / 4, dfi, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fd = 512.0 * 8 * (iters / 4) * 148.0 * 4, ff = 2.0 * 8 * dfi * 148.0 * 128;
    printf("mixed dmma %.2f TF/s + dfma %.2f TF/s = %.2f TF/s (%.3f ms)\n", fd / ms / 1e9,
           ff / ms / 1e9, (fd + ff) / ms / 1e9, ms);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
