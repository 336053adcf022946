// Max co-resident clusters per cluster size / dynamic smem on this GPU.
#include <cstdio>
__global__ void k(double* x) { extern __shared__ double s[]; if (x) x[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int kb : {60, 100, 139, 191}) {
    printf("smem %3d KB:", kb);
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = kb * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf(" %d:%d", cs, e == cudaSuccess ? n : -1);
    }
    printf("\n");
  }
}
