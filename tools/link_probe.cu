// Cycle cost of link() (ADD commit: covisibility, append, binding, counters, geometry) and
// mark_dirty for one point, one thread, warm L2 — the heads phase of an apply round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../include -I../paper_2511_02036_b200/csrc -o link_probe link_probe.cu
#include <cstdio>
#include <vector>
#include "lm_map.cuh"
using namespace lm;
__global__ void k_probe(DevMap M, int n, long long* out) {
  __shared__ PairAcc acc;
  pair_acc_init<32>(&acc, 60);
  long long best = 1ll << 60, bd = 1ll << 60;
  for (int r = 0; r < 8; ++r) {
    if (threadIdx.x == 0) {
      M.nobs[0] = n;
      M.dirty[0] = 0;
      M.gval[0] = 1;
      const long long c0 = clock64();
      link(M, 0, 63, r, &acc, true);
      const long long c1 = clock64();
      mark_dirty(M, 0);
      const long long c2 = clock64();
      best = c1 - c0 < best ? c1 - c0 : best;
      bd = c2 - c1 < bd ? c2 - c1 : bd;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = best; out[1] = bd; }
}
template <class T> T* dev(size_t n) { T* p; cudaMalloc(&p, sizeof(T) * n); cudaMemset(p, 0, sizeof(T) * n); return p; }
int main() {
  for (int n : {4, 12, 24}) {
    DevMap M = {};
    M.kf_cap = 64; M.L = 8; M.obs_cap = 1 << 16; M.mp_cap = 16;
    M.nobs = dev<int>(16); M.ocap = dev<int>(16); M.ooff = dev<int>(16); M.obs = dev<int2>(1 << 16);
    M.dirty = dev<int>(16); M.gval = dev<unsigned char>(16); M.kp_off = dev<int>(64); M.kf_id = dev<long long>(64);
    M.pos = dev<double>(48); M.C = dev<double>(64 * 3); M.klev = dev<unsigned char>(64 * 8); M.kbind = dev<int>(64 * 8);
    M.counts = dev<int>(16 * 8); M.ver = dev<int>(16); M.glo = dev<double>(16); M.ghi = dev<double>(16);
    M.gacc = dev<double>(48); M.scal = dev<int>(8); M.dirty_list = dev<int>(16); M.covis = dev<int>(64 * 64);
    std::vector<int2> o(n);
    for (int k = 0; k < n; ++k) o[k] = make_int2(k, 0);
    cudaMemcpy(M.obs, o.data(), sizeof(int2) * n, cudaMemcpyHostToDevice);
    int cap = 64; cudaMemcpy(M.ocap, &cap, 4, cudaMemcpyHostToDevice);
    std::vector<long long> ids(64); for (int k = 0; k < 64; ++k) ids[k] = k;
    cudaMemcpy(M.kf_id, ids.data(), 8 * 64, cudaMemcpyHostToDevice);
    std::vector<int> off(64); for (int k = 0; k < 64; ++k) off[k] = 8 * k;
    cudaMemcpy(M.kp_off, off.data(), 4 * 64, cudaMemcpyHostToDevice);
    double S[16]; for (int l = 0; l < 16; ++l) S[l] = 1.0; memcpy(M.S, S, sizeof S);
    long long* out = dev<long long>(2);
    k_probe<<<1, 32>>>(M, n, out);
    long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("n=%d link: %lld cycles, mark_dirty: %lld cycles (%s)\n", n, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
