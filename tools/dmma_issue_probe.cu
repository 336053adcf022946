// DMMA m8n8k4 issue rate per SMSP with DISTINCT operand registers (a GEMM-like 3x2 or 4x4
// fragment tile), 1 vs 2 vs 3 warps per SMSP.  tools/dmma_probe.cu reuses one a/b pair.
#include <cstdio>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int FM, int FN>
__global__ void k_tile(int iters, double* out) {
  double a[FM], b[FN], c[FM][FN][2];
#pragma unroll
  for (int m = 0; m < FM; ++m) a[m] = threadIdx.x * 1e-3 + m;
#pragma unroll
  for (int n = 0; n < FN; ++n) b[n] = 1.0 + n * 1e-6;
#pragma unroll
  for (int m = 0; m < FM; ++m)
#pragma unroll
    for (int n = 0; n < FN; ++n) c[m][n][0] = c[m][n][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < FM; ++m)
#pragma unroll
      for (int n = 0; n < FN; ++n) dmma(c[m][n][0], c[m][n][1], a[m], b[n]);
#pragma unroll
    for (int m = 0; m < FM; ++m) a[m] = __shfl_xor_sync(0xffffffffu, a[m], 1);  // new operands
  }
  double s = 0;
#pragma unroll
  for (int m = 0; m < FM; ++m)
#pragma unroll
    for (int n = 0; n < FN; ++n) s += c[m][n][0] + c[m][n][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int FM, int FN>
void run(int warps_per_block, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  k_tile<FM, FN><<<148, warps_per_block * 32>>>(10, out);
  cudaEventRecord(e0);
  k_tile<FM, FN><<<148, warps_per_block * 32>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * FM * FN * iters * 148.0 * warps_per_block;
  printf("tile %dx%d, %d warps/SM (%d per SMSP): %.2f TFLOP/s\n", FM, FN, warps_per_block,
         warps_per_block / 4, flops / ms / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 24);
  for (int w : {4, 8, 12}) {
    run<3, 1>(w, out);  // the all-SM chain kernel's tile (3 row strips x 8 columns)
    run<2, 1>(w, out);
    run<1, 1>(w, out);
    run<3, 2>(w, out);
    run<2, 2>(w, out);
    run<4, 4>(w, out);
    run<4, 3>(w, out);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
