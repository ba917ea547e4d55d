// Latency constants of the single-CTA chains on this GPU: dependent global load (L2 hit),
// dependent global atomicAdd / atomicExch (returning), shared atomic, __syncthreads (1024 threads),
// globaltimer resolution. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_chain_load(int* p, int n, long long* out) {
  int i = 0;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) i = p[i];
  long long t1 = clock64();
  out[0] = (t1 - t0) / n;
  out[1] = i;
}
__global__ void k_chain_atomic(int* p, int n, long long* out) {
  int i = 0;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) i = atomicAdd(&p[i & 1023], 1) & 1023;
  long long t1 = clock64();
  out[0] = (t1 - t0) / n;
  out[1] = i;
}
__global__ void k_chain_exch(int* p, int n, long long* out) {
  int i = 0;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) i = atomicExch(&p[i & 1023], i + 1) & 1023;
  long long t1 = clock64();
  out[0] = (t1 - t0) / n;
  out[1] = i;
}
__global__ void k_sync(int n, long long* out) {
  __shared__ int x;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) x = k;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}
__global__ void k_contended(int* p, int n, long long* out) {  // all threads of a CTA atomicAdd one word
  long long t0 = clock64();
  int v = 0;
  for (int k = 0; k < n; ++k) v += atomicAdd(&p[0], 1);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / n; out[1] = v; }
}
__global__ void k_gtimer(long long* out) {
  unsigned long long a, b;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b)); } while (b == a);
  out[0] = (long long)(b - a);
}
__global__ void k_cluster_sync(int n, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / n;
}
int main() {
  int* p; long long* o; long long h[2];
  cudaMalloc(&p, 1 << 24); cudaMalloc(&o, 64);
  int* hp = new int[1 << 22];
  for (int i = 0; i < (1 << 22); ++i) hp[i] = (int)((i * 2654435761u + 12345u) % (1u << 20));  // random chain in 4 MB
  cudaMemcpy(p, hp, 4 << 20, cudaMemcpyHostToDevice);
  k_chain_load<<<1, 1>>>(p, 1 << 14, o); k_chain_load<<<1, 1>>>(p, 1 << 14, o);
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("dependent global load (L2-resident 4MB): %lld cycles\n", h[0]);
  {  // 64 MB random chain (L2-resident on a 126 MB L2, spread over both dies' slices)
    int* q; const int N = 1 << 24; cudaMalloc(&q, sizeof(int) * N);
    int* hq = new int[N];
    for (int i = 0; i < N; ++i) hq[i] = (int)((i * 2654435761u + 7u) % (unsigned)N);
    cudaMemcpy(q, hq, sizeof(int) * N, cudaMemcpyHostToDevice);
    k_chain_load<<<1, 1>>>(q, 1 << 14, o); k_chain_load<<<1, 1>>>(q, 1 << 14, o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("dependent global load (64MB chain): %lld cycles\n", h[0]);
    for (int sm = 0; sm < 2; ++sm) {}
    cudaFree(q); delete[] hq;
  }
  cudaMemset(p, 0, 1 << 12);
  k_chain_atomic<<<1, 1>>>(p, 1 << 12, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("dependent global atomicAdd (returning): %lld cycles\n", h[0]);
  k_chain_exch<<<1, 1>>>(p, 1 << 12, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("dependent global atomicExch: %lld cycles\n", h[0]);
  for (int t : {32, 256, 1024}) {
    k_sync<<<1, t>>>(1 << 12, o); cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads loop, %d threads: %lld cycles\n", t, h[0]);
  }
  cudaMemset(p, 0, 4);
  k_contended<<<1, 1024>>>(p, 64, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("1024 threads atomicAdd one word, per iteration: %lld cycles\n", h[0]);
  for (int cs : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(1024);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cluster_sync, 1 << 12, o); cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost);
    printf("cluster.sync, %d CTAs x 1024 threads: %lld cycles (%s)\n", cs, h[0], cudaGetErrorString(cudaGetLastError()));
  }
  k_gtimer<<<1, 1>>>(o); cudaMemcpy(h, o, 8, cudaMemcpyDeviceToHost); printf("globaltimer tick: %lld ns\n", h[0]);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
  return 0;
}
