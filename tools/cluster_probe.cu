// Microbenchmark: per-step cost of the recurrence building blocks on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int steps) {
  cg::cluster_group cl = cg::this_cluster();
  for (int s = 0; s < steps; ++s) cl.sync();
}

__global__ void k_arrive_wait_relaxed(int steps) {
  for (int s = 0; s < steps; ++s) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::);
    asm volatile("barrier.cluster.wait.aligned;\n" ::);
  }
}

// push: each of `outs` threads pushes one double into every CTA of the cluster
__global__ void k_push(int steps, int outs) {
  extern __shared__ double xs[];
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks();
  cl.sync();
  for (int s = 0; s < steps; ++s) {
    double* nxt = xs + ((s + 1) & 1) * 4096;
    if (threadIdx.x < outs) {
      const int slot = cl.block_rank() * outs + threadIdx.x;
      for (int q = 0; q < cs; ++q) *cl.map_shared_rank(nxt + slot, q) = (double)s;
    }
    cl.sync();
  }
}

// pull: after the barrier each thread reads `per` doubles from peers' smem
__global__ void k_pull(int steps, int outs) {
  extern __shared__ double xs[];
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks();
  double acc = 0;
  cl.sync();
  for (int s = 0; s < steps; ++s) {
    double* cur = xs + (s & 1) * 4096;
    if (threadIdx.x < outs) cur[threadIdx.x] = (double)s;
    cl.sync();
    for (int q = 0; q < cs; ++q) {
      const double* rp = cl.map_shared_rank(cur, q);
      for (int i = threadIdx.x; i < outs; i += blockDim.x) acc += rp[i];
    }
  }
  cl.sync();
  if (acc == 12345.0) xs[0] = acc;
}

// L2: write outs values to global, barrier, read cs*outs values back with ldcg
__global__ void k_l2(int steps, int outs, double* buf) {
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks();
  const int cid = blockIdx.x / cs;
  double* base = buf + (size_t)cid * 2 * cs * outs;
  double acc = 0;
  for (int s = 0; s < steps; ++s) {
    double* cur = base + (s & 1) * cs * outs;
    if (threadIdx.x < outs) cur[cl.block_rank() * outs + threadIdx.x] = (double)s;
    cl.sync();
    for (int i = threadIdx.x; i < cs * outs; i += blockDim.x) acc += __ldcg(cur + i);
  }
  if (acc == 12345.0) buf[0] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms;
}

template <class K, class... Args>
void launch(K kern, int cs, int nclusters, size_t smem, Args... args) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * nclusters);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) printf("launch err cs=%d %s\n", cs, cudaGetErrorString(e));
}

int main() {
  const int steps = 2000;
  double* buf;
  cudaMalloc(&buf, 64 << 20);
  setvbuf(stdout, NULL, _IONBF, 0);
  printf("start\n");
  for (int cs : {4, 8, 13, 16}) {
    printf("cs %d\n", cs);
    const int ncl = 104 / cs > 0 ? 104 / cs : 1;
    float t1 = timeit([&] { launch(k_sync, cs, ncl, 0, steps); });
    float t2 = timeit([&] { launch(k_arrive_wait_relaxed, cs, ncl, 0, steps); });
    float t3 = timeit([&] { launch(k_push, cs, ncl, 2 * 4096 * 8, steps, 192); });
    float t4 = timeit([&] { launch(k_pull, cs, ncl, 2 * 4096 * 8, steps, 192); });
    float t5 = timeit([&] { launch(k_l2, cs, ncl, 0, steps, 192, buf); });
    printf("cs=%2d clusters=%2d  sync %.3f us  relaxed %.3f us  push %.3f us  pull %.3f us  l2 %.3f us per step\n",
           cs, ncl, t1 * 1e3 / steps, t2 * 1e3 / steps, t3 * 1e3 / steps, t4 * 1e3 / steps,
           t5 * 1e3 / steps);
  }
  return 0;
}
