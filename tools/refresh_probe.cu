// Cycle cost of one warp's representative-descriptor refresh (refresh_rep_warp) for a point
// with n observations, in isolation (one warp, warm L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../include -I../paper_2511_02036_b200/csrc -o refresh_probe refresh_probe.cu
#include <cstdio>
#include <vector>
#include "lm_map.cuh"
using namespace lm;
__global__ void k_probe(DevMap M, int reps, long long* out) {
  const int lane = threadIdx.x & 31;
  long long best = 1ll << 60;
  for (int r = 0; r < reps; ++r) {
    const long long c0 = clock64();
    refresh_rep_warp(M, 0, lane);
    __syncwarp();
    const long long c1 = clock64();
    best = c1 - c0 < best ? c1 - c0 : best;
  }
  if (lane == 0) out[0] = best;
}
int main() {
  for (int n : {8, 16, 24, 32, 48, 64}) {
    DevMap M = {};
    const int nkf = 64;
    std::vector<int2> obs(n);
    std::vector<long long> kfid(nkf);
    std::vector<int> kpoff(nkf);
    std::vector<uint4> desc(2 * nkf * 4);
    for (int k = 0; k < nkf; ++k) { kfid[k] = 1000 - 7 * k; kpoff[k] = 4 * k; }
    for (int i = 0; i < n; ++i) obs[i] = make_int2((i * 37) % nkf, i % 4);
    unsigned s = 12345;
    for (auto& d : desc) { s = s * 1664525u + 1013904223u; d.x = s; s = s * 1664525u + 1013904223u; d.y = s;
                           s = s * 1664525u + 1013904223u; d.z = s; s = s * 1664525u + 1013904223u; d.w = s; }
    int nobs = n, ooff = 0;
    int2* d_obs; long long* d_kf; int* d_off; uint4* d_desc; int* d_n; int* d_oo; uint4* d_rep; int* d_scal; long long* d_out;
    cudaMalloc(&d_obs, sizeof(int2) * n); cudaMalloc(&d_kf, 8 * nkf); cudaMalloc(&d_off, 4 * nkf);
    cudaMalloc(&d_desc, sizeof(uint4) * desc.size()); cudaMalloc(&d_n, 4); cudaMalloc(&d_oo, 4); cudaMalloc(&d_rep, 32);
    cudaMalloc(&d_scal, 64); cudaMalloc(&d_out, 8);
    cudaMemcpy(d_obs, obs.data(), sizeof(int2) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(d_kf, kfid.data(), 8 * nkf, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off, kpoff.data(), 4 * nkf, cudaMemcpyHostToDevice);
    cudaMemcpy(d_desc, desc.data(), sizeof(uint4) * desc.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_n, &nobs, 4, cudaMemcpyHostToDevice); cudaMemcpy(d_oo, &ooff, 4, cudaMemcpyHostToDevice);
    M.obs = d_obs; M.kf_id = d_kf; M.kp_off = d_off; M.kdesc = d_desc; M.nobs = d_n; M.ooff = d_oo; M.rep = d_rep;
    M.scal = d_scal;
    k_probe<<<1, 32>>>(M, 20, d_out);
    long long cyc = 0;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    printf("n=%d refresh_rep_warp: %lld cycles (%s)\n", n, cyc, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
