// Which hardware warp slots (%warpid) do the warps of co-resident 6-warp CTAs get?
// SMSP = %warpid % 4; prints, per SM, the number of warps per SMSP.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void probe(int* out, int spin) {
  extern __shared__ double sm[];
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if ((threadIdx.x & 31) == 0) {
    int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    out[2 * w] = smid;
    out[2 * w + 1] = wid;
  }
  // keep the CTA resident so that the second CTA of the SM must co-reside
  long long t0 = clock64();
  while (clock64() - t0 < spin) sm[threadIdx.x] += 1.0;
}
int main(int argc, char** argv) {
  int threads = argc > 1 ? atoi(argv[1]) : 192, ctas = argc > 2 ? atoi(argv[2]) : 285;
  int smem = argc > 3 ? atoi(argv[3]) : 60 * 1024;
  int nw = ctas * threads / 32;
  int* d;
  cudaMalloc(&d, sizeof(int) * 2 * nw);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<ctas, threads, smem>>>(d, 2000000);
  cudaDeviceSynchronize();
  std::vector<int> h(2 * nw);
  cudaMemcpy(h.data(), d, sizeof(int) * 2 * nw, cudaMemcpyDeviceToHost);
  int cnt[160][4] = {};
  for (int w = 0; w < nw; ++w) cnt[h[2 * w]][h[2 * w + 1] & 3]++;
  int hist[16] = {};
  for (int s = 0; s < 148; ++s) {
    int mx = 0;
    for (int q = 0; q < 4; ++q) mx = cnt[s][q] > mx ? cnt[s][q] : mx;
    hist[mx]++;
    if (s < 6) printf("sm %d: %d %d %d %d\n", s, cnt[s][0], cnt[s][1], cnt[s][2], cnt[s][3]);
  }
  for (int i = 0; i < 16; ++i)
    if (hist[i]) printf("max warps on one SMSP = %d: %d SMs\n", i, hist[i]);
  printf("first CTAs' slots:");
  for (int w = 0; w < 12; ++w) printf(" (%d,%d)", h[2 * w], h[2 * w + 1]);
  printf("\n");
  return 0;
}
