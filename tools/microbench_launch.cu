// Launch floor on this GPU: CUDA-event time per launch of an (almost) empty kernel, plain vs
// thread-block-cluster launches, with the shared-memory footprint of k_small_fused.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbl tools/microbench_launch.cu && tools/mbl
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_empty(int* o) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && sm[5] == 7) o[blockIdx.x] = 1;
}
__global__ void k_empty_cl(int* o) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  cg::this_cluster().sync();
  if (threadIdx.x == 0 && sm[5] == 7) o[blockIdx.x] = 1;
}
static float run(int ctas, int cl, size_t smem, bool graph) {
  int* o; cudaMalloc(&o, 4096);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = cl > 0 ? 1 : 0;
  auto kern = cl > 0 ? k_empty_cl : k_empty;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int N = 200;
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, o);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    cudaEventRecord(e0, st);
    if (graph) cudaGraphLaunch(ge, st);
    else for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, o);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1000.f / N;
}
int main() {
  const size_t sm[2] = {16 * 1024, 160 * 1024};
  for (int s = 0; s < 2; ++s)
    for (int cl : {0, 4, 8, 16})
      printf("ctas 16 cluster %2d smem %3zu KB: stream %.2f us/launch, graph %.2f us/launch\n", cl, sm[s] / 1024,
             run(16, cl, sm[s], false), run(16, cl, sm[s], true));
  return 0;
}
