// lm_b200.cu -- C ABI of the B200 local-mapping hot path (see include/lm_b200.h).
//
// Host responsibilities only: arena allocation, keyframe staging (one pinned->device copy
// and one scatter/grid kernel per keyframe), slot bookkeeping, kernel launches on the
// context's stream, and exports. No hot-path arithmetic runs on the host: the per-keyframe
// pose tables (R, C, P = K[R|t]) are computed here once at staging with the same
// __host__ __device__ code the kernels use (lm_math.cuh).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstddef>
#include <cmath>
#include <string>
#include <unordered_map>
#include <vector>

#include "lm_kernels.cuh"
#include "lm_audit.cuh"

using namespace lm;

namespace {

constexpr int kRing = 64;       // step-argument ring entries
constexpr int kMaxBatch = 128;  // maps per batched step
constexpr int kStageRing = 4;   // keyframe staging buffers

struct StageHdr {
  int slot, n, kp_off, nx, ny;
  double cs;
  long long kf_id;
  double q[4], R[9], t[3], C[3], P[12], cam[6];
};

struct HostMap {
  DevMap d{};
  lm_map_caps caps{};
  std::unordered_map<long long, int> slot_of;
  std::vector<int> state;  // host mirror of kf_state
  std::vector<char> res;   // host mirror of kf_res (DeviceStore residency)
  std::vector<char> prebound;  // staged with pre-bound slots (insert must report their errors)
  std::vector<int> kp_n, kp_off;
  std::vector<long long> ids;
  int n_slots = 0, kp_head = 0, resident = 0;
  std::vector<void*> allocs;
  lm_step_stats* d_stats = nullptr;
  lm_step_stats* d_totals = nullptr;
  int* d_result = nullptr;  // single-op results
  void* d_io = nullptr;     // single-op input/output scratch (grown on demand)
  size_t io_bytes = 0;
};

}  // namespace

struct lm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<HostMap*> maps;
  DevMap* d_maps = nullptr;
  int d_maps_cap = 0;
  lm_step_stats** d_totals = nullptr;  // per map running totals (device pointers)
  StepArgs* h_args = nullptr;  // pinned [kRing * kMaxBatch]
  StepArgs* d_args = nullptr;
  cudaEvent_t args_ev[kRing];
  bool args_used[kRing];
  int ring_pos = 0;
  cudaStream_t stage_stream = nullptr;  // keyframe staging (H2D + k_stage), overlapping the steps
  int last_stage_b = -1;                // ring entry of the latest staging
  bool stage_unjoined = false;          // a staging the step stream has not waited for yet
  unsigned char* h_stage[kStageRing];
  unsigned char* d_stage[kStageRing];
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev[kStageRing];
  bool stage_used[kStageRing];
  long long stage_pos = 0;
  lm_step_stats* h_stats = nullptr;  // pinned [kMaxBatch]
  unsigned char* h_io = nullptr;     // pinned scratch of single-call list operations (grown on demand)
  size_t h_io_bytes = 0;
  std::string err;
  long long launches = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  bool prof = false;
  int apply_cluster = 16;               // CTAs per map of the forward-apply cluster (LM_APPLY_CLUSTER)
  int cull_cluster = 8;                 // CTAs per map of the recent-point cull cluster (LM_CULL_CLUSTER)
  int rev_cluster = 8;                  // CTAs per map of the reverse walk (LM_REV_CLUSTER; 1 = CTA 0 alone)
  int tri_slices = 4;                   // k_tri CTAs per neighbour (LM_TRI_SLICES)
  int rev_wide = 1 | 1 << 8;            // k_fuse_rev cluster-wide thresholds (LM_REV_WIDE="direct,other")
  int refresh_blocks = 148;             // k_fuse_refresh grid (x) (LM_REFRESH_BLOCKS)
  int post_blocks = 148;                // k_fuse_post grid (x), <= POST_BLOCKS (LM_POST_BLOCKS)
  // programmatic dependent launch of the step kernels (LM_PDL=0/1 overrides): on for
  // single-session launches; off for batches, whose concurrent stream groups lose SMs to
  // successor CTAs parked in griddepcontrol.wait (C5: 16.2k -> 11.6k KF/s with it)
  int pdl = -1;
  bool pdl_now = false;                 // this launch sequence
  std::vector<cudaEvent_t> prof_pool;   // free events
  std::vector<std::vector<cudaEvent_t>> prof_steps;  // 9 boundary events per step
};

static int fail(lm_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, LM_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())

template <class T>
static int arena(lm_ctx* ctx, HostMap* m, T** p, size_t count) {
  void* q = nullptr;
  CU(cudaMalloc(&q, count * sizeof(T) + 16));
  CU(cudaMemsetAsync(q, 0, count * sizeof(T) + 16, ctx->stream));
  m->allocs.push_back(q);
  *p = (T*)q;
  return LM_OK;
}

// Keyframes are staged on their own stream (lm_kf_stage), so the upload and scatter of the
// next keyframe overlap the step already queued. Every other entry point (steps included)
// first orders the step stream after all staging issued so far (join = true): nothing on the
// step stream ever sees a keyframe half staged.
static int join_staging(lm_ctx* ctx) {
  if (ctx->stage_unjoined) {
    const cudaError_t e = cudaStreamWaitEvent(ctx->stream, ctx->stage_ev[ctx->last_stage_b], 0);
    if (e != cudaSuccess) return fail(ctx, LM_ERR_CUDA, "join staging: %s", cudaGetErrorString(e));
    ctx->stage_unjoined = false;
  }
  return LM_OK;
}

static int check_map(lm_ctx* ctx, int32_t map, HostMap** out, bool join = true) {
  if (!ctx) return LM_ERR_INVALID_ARGUMENT;
  if (map < 0 || map >= (int)ctx->maps.size() || !ctx->maps[map])
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown map %d", map);
  *out = ctx->maps[map];
  return join ? join_staging(ctx) : LM_OK;
}

static int slot_of(lm_ctx* ctx, HostMap* m, long long kf_id, int* slot, bool need_live) {
  auto it = m->slot_of.find(kf_id);
  if (it == m->slot_of.end()) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown keyframe %lld", kf_id);
  *slot = it->second;
  if (need_live && m->state[*slot] != KF_LIVE)
    return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld is not live", kf_id);
  return LM_OK;
}

static int upload_maps(lm_ctx* ctx) {
  const int n = (int)ctx->maps.size();
  if (n > ctx->d_maps_cap) {
    if (ctx->d_maps) CU(cudaFree(ctx->d_maps));
    ctx->d_maps_cap = n < 16 ? 16 : 2 * n;
    CU(cudaMalloc(&ctx->d_maps, sizeof(DevMap) * ctx->d_maps_cap));
  }
  std::vector<DevMap> h(n);
  for (int i = 0; i < n; ++i) h[i] = ctx->maps[i] ? ctx->maps[i]->d : DevMap{};
  CU(cudaMemcpyAsync(ctx->d_maps, h.data(), sizeof(DevMap) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->d_totals) CU(cudaFree(ctx->d_totals));
  CU(cudaMalloc(&ctx->d_totals, sizeof(lm_step_stats*) * n));
  std::vector<lm_step_stats*> tp(n);
  for (int i = 0; i < n; ++i) tp[i] = ctx->maps[i] ? ctx->maps[i]->d_totals : nullptr;
  CU(cudaMemcpyAsync(ctx->d_totals, tp.data(), sizeof(lm_step_stats*) * n, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return LM_OK;
}

// scatter a staged keyframe into the arenas and build its cell grid
__global__ void __launch_bounds__(1024) k_stage(DevMap M, const unsigned char* buf) {
  const StageHdr* h = (const StageHdr*)buf;
  const int n = h->n, off = h->kp_off, slot = h->slot;
  const double* u = (const double*)(buf + sizeof(StageHdr));
  const double* v = u + n;
  const uint4* desc = (const uint4*)(v + n);
  const int* bind = (const int*)(desc + 2 * n);
  const unsigned char* lev = (const unsigned char*)(bind + n);
  __shared__ int cnt[GRID_CELLS];
  __shared__ int sh[32];
  if (threadIdx.x == 0) {
    M.kf_id[slot] = h->kf_id;
    M.kp_off[slot] = off;
    M.kp_n[slot] = n;
    for (int k = 0; k < 4; ++k) M.q[4 * slot + k] = h->q[k];
    for (int k = 0; k < 9; ++k) M.R[9 * slot + k] = h->R[k];
    for (int k = 0; k < 3; ++k) M.t[3 * slot + k] = h->t[k];
    for (int k = 0; k < 3; ++k) M.C[3 * slot + k] = h->C[k];
    for (int k = 0; k < 12; ++k) M.P[12 * slot + k] = h->P[k];
    for (int k = 0; k < 6; ++k) M.cam[6 * slot + k] = h->cam[k];
    M.g_cs[slot] = h->cs;
    M.g_nx[slot] = h->nx;
    M.g_ny[slot] = h->ny;
    M.kf_state[slot] = KF_STAGED;
  }
  const int nx = h->nx, ny = h->ny, nc = nx * ny;
  const double cs = h->cs;
  for (int c = threadIdx.x; c < nc; c += 1024) cnt[c] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += 1024) {
    M.ku[off + i] = u[i];
    M.kv[off + i] = v[i];
    M.kdesc[2 * (off + i)] = desc[2 * i];
    M.kdesc[2 * (off + i) + 1] = desc[2 * i + 1];
    M.kbind[off + i] = bind[i];
    M.klev[off + i] = lev[i];
    const double fx = floor(u[i] / cs), fy = floor(v[i] / cs);
    int cx = fx == fx ? (fx < 0 ? 0 : (fx > nx - 1 ? nx - 1 : (int)fx)) : 0;
    int cy = fy == fy ? (fy < 0 ? 0 : (fy > ny - 1 ? ny - 1 : (int)fy)) : 0;
    atomicAdd(&cnt[cy * nx + cx], 1);
  }
  __syncthreads();
  // exclusive scan of cell counts (chunked block scan)
  int* cst = M.cell_start + (size_t)slot * (GRID_CELLS + 1);
  int run = 0;
  for (int b0 = 0; b0 < nc; b0 += 1024) {
    const int c = b0 + threadIdx.x;
    const int x = c < nc ? cnt[c] : 0;
    int tot;
    const int at = block_excl_scan<1024>(x, sh, tot);
    if (c < nc) {
      cst[c] = run + at;
      cnt[c] = run + at;  // cursor
    }
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cst[nc] = run;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += 1024) {
    const double fx = floor(u[i] / cs), fy = floor(v[i] / cs);
    int cx = fx == fx ? (fx < 0 ? 0 : (fx > nx - 1 ? nx - 1 : (int)fx)) : 0;
    int cy = fy == fy ? (fy < 0 ? 0 : (fy > ny - 1 ? ny - 1 : (int)fy)) : 0;
    const int at = atomicAdd(&cnt[cy * nx + cx], 1);
    M.cell_items[off + at] = i;  // local keypoint index
  }
}

// ------------------------------------------------------------------- single-op map kernel
enum MapOp { OP_NEW = 1, OP_OBS_ADD, OP_OBS_ERASE, OP_KILL, OP_REPLACE, OP_SET_COUNTS, OP_KF_KILL, OP_NEIGHBORS,
             OP_REFRESH, OP_APPLY, OP_TARGETS, OP_FUSE_PASS, OP_CULL, OP_SET_POSE, OP_PATCH_POS, OP_UPLOAD, OP_EVICT,
             OP_MP_GET, OP_BOUND, OP_IMPORT_POINTS, OP_LEDGER_ADD, OP_CORRUPT, OP_KF_CULL, OP_GEO_ALL };

// kill_keyframe (mapmodel.py:275-283), whole block. The reference erases this keyframe's
// observation of every bound point in id order; each erase touches only its own point (list,
// counters, a possible kill_point) plus commutative covisibility decrements, and a point is
// bound at most once per keyframe, so the erases are independent: thread per keypoint.
__device__ void kill_keyframe_block(const DevMap& M, int slot) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int off = M.kp_off[slot], n = M.kp_n[slot];
  __syncthreads();
  for (int i = tid; i < n; i += nth) {
    const int mp = M.kbind[off + i];
    if (mp < 0) continue;
    const int k = M.alive[mp] ? obs_find(M, mp, slot) : -1;
    if (k >= 0) {
      unlink_at(M, mp, k);
      if (M.nobs[mp] < M.min_obs_keep) kill_point(M, mp);
      else mark_dirty(M, mp);
    } else {
      M.kbind[off + i] = -1;
    }
  }
  __syncthreads();
  for (int s = tid; s < M.kf_cap; s += nth) {  // graph.drop_keyframe
    M.covis[(size_t)slot * M.kf_cap + s] = 0;
    M.covis[(size_t)s * M.kf_cap + slot] = 0;
  }
  if (tid == 0) M.kf_state[slot] = KF_DEAD;
  __syncthreads();
}

// packed single-point record of OP_MP_GET (lm_mp_get), followed by nobs int2 (slot, kp)
struct PointRec {
  double pos[3];
  uint4 rep[2];
  long long first_kf;
  int alive, found, visible, nobs;
  int counts[LMAX];
};

struct OpArgs {
  int op;
  int a, b, c;        // ids / slots / kp
  int n;              // count
  double pos[3];
  unsigned char desc[32];
  long long first_kf;
  int found, visible;
  lm_fuse_cfg fc;
  lm_cull_cfg cc;
  int processed;
  int n_slots;
  double pose[4 + 9 + 3 + 3 + 12];  // OP_SET_POSE: q, R, t, C, P
  void* buf;                        // OP_PATCH_POS / OP_MP_GET / OP_BOUND / OP_IMPORT_POINTS: io scratch
  long long v0, v1;                 // OP_LEDGER_ADD: naive bytes, small-transfer bytes
  double kc_ratio;                  // OP_KF_CULL: CullConfig redundancy_ratio,
  int kc_min_obs, kc_tol;           //   min_redundant_observers, scale_tolerance_levels
};

__global__ void __launch_bounds__(1024) k_op(DevMap* maps, int map, OpArgs A, int* res) {
  const DevMap& M = maps[map];
  extern __shared__ __align__(16) int dyn[];
  __shared__ int sh[32];
  __shared__ int out_nb[1024];
  const int tid = threadIdx.x;
  switch (A.op) {
    case OP_NEW: {
      if (tid) return;
      const int id = M.scal[SC_NEXT_ID];
      if (id >= M.mp_cap) {
        res[0] = LM_ERR_CAPACITY;
        return;
      }
      M.scal[SC_NEXT_ID] = id + 1;
      for (int k = 0; k < 3; ++k) M.pos[3 * id + k] = A.pos[k];
      uint4 r[2];
      memcpy(r, A.desc, 32);
      M.rep[2 * id] = r[0];
      M.rep[2 * id + 1] = r[1];
      M.alive[id] = 1;
      M.found[id] = 1;
      M.visible[id] = 1;
      M.first_kf[id] = A.first_kf;
      M.nobs[id] = 0;
      M.ocap[id] = 0;
      M.ooff[id] = 0;
      M.gval[id] = 0;
      M.dirty[id] = 0;
      res[0] = LM_OK;
      res[1] = id;
      return;
    }
    case OP_OBS_ADD: {
      if (tid) return;
      const int mp = A.a, slot = A.b, kp = A.c;
      if (mp < 0 || mp >= M.scal[SC_NEXT_ID]) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      if (!M.alive[mp]) { res[0] = LM_ERR_INVALID_STATE; return; }
      if (kp < 0 || kp >= M.kp_n[slot]) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      if (M.kbind[M.kp_off[slot] + kp] >= 0) { res[0] = LM_ERR_SLOT_CONFLICT; res[1] = M.kbind[M.kp_off[slot] + kp]; return; }
      if (obs_find(M, mp, slot) >= 0) { res[0] = LM_ERR_SLOT_CONFLICT; res[1] = -2; return; }
      link(M, mp, slot, kp);
      mark_dirty(M, mp);
      res[0] = M.scal[SC_ERR] ? M.scal[SC_ERR] : LM_OK;
      return;
    }
    case OP_OBS_ERASE: {
      if (tid) return;
      const int mp = A.a, slot = A.b;
      if (mp < 0 || mp >= M.scal[SC_NEXT_ID]) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      if (!M.alive[mp]) { res[0] = LM_ERR_INVALID_STATE; return; }
      const int k = obs_find(M, mp, slot);
      if (k < 0) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      unlink_at(M, mp, k);
      if (M.nobs[mp] < M.min_obs_keep) kill_point(M, mp);
      else mark_dirty(M, mp);
      res[0] = LM_OK;
      return;
    }
    case OP_KILL: {
      if (tid) return;
      const int mp = A.a;
      if (mp < 0 || mp >= M.scal[SC_NEXT_ID]) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      if (!M.alive[mp]) { res[0] = LM_ERR_INVALID_STATE; return; }
      kill_point(M, mp);
      res[0] = LM_OK;
      return;
    }
    case OP_REPLACE: {
      if (tid) return;
      const int lo = A.a, wi = A.b;
      if (lo == wi || lo < 0 || wi < 0 || lo >= M.scal[SC_NEXT_ID] || wi >= M.scal[SC_NEXT_ID]) {
        res[0] = LM_ERR_INVALID_ARGUMENT;
        return;
      }
      if (!M.alive[lo] || !M.alive[wi]) { res[0] = LM_ERR_INVALID_STATE; return; }
      if (M.nobs[lo] > M.nobs[wi]) { res[0] = LM_ERR_INVALID_ARGUMENT; return; }
      res[1] = replace_point(M, lo, wi);
      res[0] = LM_OK;
      return;
    }
    case OP_SET_COUNTS: {
      if (tid) return;
      M.found[A.a] = A.found;
      M.visible[A.a] = A.visible;
      res[0] = LM_OK;
      return;
    }
    case OP_KF_KILL: {  // kill_keyframe mapmodel.py:275-283
      kill_keyframe_block(M, A.a);
      if (tid == 0) res[0] = LM_OK;
      return;
    }
    case OP_KF_CULL: {  // cull_keyframes culling.py:127-154 with is_redundant_* 60-117
      // candidates (slots, ascending kf id, deduplicated, slot of kf 0 dropped) in A.buf;
      // removed slots appended after them. Sequential over candidates: a removal is visible
      // to every later candidate's check.
      int* cand = (int*)A.buf;
      int* removed = cand + A.n;
      __shared__ int nrem;
      if (tid == 0) nrem = 0;
      for (int c = 0; c < A.n; ++c) {
        const int slot = cand[c];
        __syncthreads();
        if (M.kf_state[slot] != KF_LIVE) continue;  // (uniform)
        const int off = M.kp_off[slot], n = M.kp_n[slot];
        int rp = 0, cs = 0;
        for (int i = tid; i < n; i += 1024) {
          const int mp = M.kbind[off + i];
          if (mp < 0 || !M.alive[mp]) continue;
          ++cs;
          // counter prefix up to the keypoint's level + tolerance (is_redundant_fast), minus
          // the keyframe's own observation (== the baseline's observation-list walk)
          int lim = (int)M.klev[off + i] + A.kc_tol;
          lim = lim > M.L - 1 ? M.L - 1 : lim;
          int pre = 0;
          for (int l = 0; l <= lim; ++l) pre += M.counts[(size_t)mp * M.L + l];
          rp += pre - 1 >= A.kc_min_obs;
        }
        rp = block_sum<1024>(rp, sh);
        cs = block_sum<1024>(cs, sh);
        const bool redundant = cs > 0 && (double)rp >= A.kc_ratio * (double)cs;
        if (!redundant) continue;  // (uniform)
        kill_keyframe_block(M, slot);
        if (tid == 0) {
          if (M.kf_res[slot]) {  // store.evict_keyframe when resident
            M.kf_res[slot] = 0;
            M.ledger[LG_EVICT] += 1;
          }
          removed[nrem++] = slot;
        }
      }
      __syncthreads();
      if (tid == 0) {
        res[0] = LM_OK;
        res[1] = nrem;
      }
      return;
    }
    case OP_NEIGHBORS: {
      unsigned long long* sh_key = (unsigned long long*)dyn;
      int* sh_slot = (int*)(sh_key + M.kf_cap);
      const int got = ranked_neighbors<1024>(M, A.a, A.n, sh_slot, sh_key, out_nb, A.n_slots);
      for (int k = tid; k < got; k += 1024) res[2 + k] = out_nb[k];
      if (tid == 0) {
        res[0] = LM_OK;
        res[1] = got;
      }
      return;
    }
    case OP_REFRESH: {
      refresh_all<1024>(M);
      if (tid == 0) res[0] = M.scal[SC_ERR];
      return;
    }
    case OP_APPLY: {
      __shared__ int c[3];
      __shared__ PairAcc acc;
      if (tid < 3) c[tid] = 0;
      pair_acc_init<1024>(&acc, A.n_slots - 1);
      apply_block<1024>(M, M.s.acts, A.n, c, sh, &acc);
      pair_acc_flush<1024>(M, &acc);
      if (tid == 0) {
        res[0] = M.scal[SC_ERR];
        res[1] = c[0];
        res[2] = c[1];
        res[3] = c[2];
      }
      return;
    }
    case OP_TARGETS: {
      unsigned long long* sh_key = (unsigned long long*)dyn;
      int* sh_slot = (int*)(sh_key + M.kf_cap);
      const int T = fusion_targets<1024>(M, A.a, A.fc.n1, A.fc.n2, A.n_slots, sh_slot, sh_key);
      if (tid == 0) {
        res[0] = LM_OK;
        res[1] = T;
      }
      return;
    }
    case OP_FUSE_PASS: {
      int nvis = 0;
      const int na = gather_pass<1024>(M, A.fc, A.n, A.a, tgt_global(M, A.a), false, sh, &nvis);
      if (tid == 0) {
        res[0] = M.scal[SC_ERR];
        res[1] = na;
        res[2] = nvis;
      }
      return;
    }
    case OP_SET_POSE: {  // LBA pose write-back (localba.py:571-574): tables + geometry caches
      const int slot = A.a;
      if (tid == 0) {
        for (int k = 0; k < 4; ++k) M.q[4 * slot + k] = A.pose[k];
        for (int k = 0; k < 9; ++k) M.R[9 * slot + k] = A.pose[4 + k];
        for (int k = 0; k < 3; ++k) M.t[3 * slot + k] = A.pose[13 + k];
        for (int k = 0; k < 3; ++k) M.C[3 * slot + k] = A.pose[16 + k];
        for (int k = 0; k < 12; ++k) M.P[12 * slot + k] = A.pose[19 + k];
      }
      // every point observed here has a ray from this camera centre in its cached
      // _point_geometry sums (fusion.py:57-94) and a cached hit: both stale now. A point
      // observes a keyframe at most once, so each is touched by one thread.
      // Invariant kept for the stages: a live point's geometry cache is valid unless the point
      // is listed dirty (the refresh recomputes it then); several gather threads may read one
      // point's cache concurrently, so a stale-but-clean cache must never be left behind.
      const int off = M.kp_off[slot], n = M.kp_n[slot];
      __syncthreads();  // (thread 0's pose writes before any geometry term reads them)
      for (int i = tid; i < n; i += 1024) {
        const int mp = M.kbind[off + i];
        if (mp >= 0) {
          M.ver[mp] += 1;
          if (M.alive[mp] && !M.dirty[mp]) geo_full(M, mp);
          else M.gval[mp] = 0;
        }
      }
      if (tid == 0) res[0] = LM_OK;
      return;
    }
    case OP_PATCH_POS: {  // LBA position write-back: buf = n x (int id, pad, double xyz)
      const int n = A.n;
      const char* b = (const char*)A.buf;
      for (int k = tid; k < n; k += 1024) {
        const int mp = *(const int*)(b + 32 * (size_t)k);
        const double* x = (const double*)(b + 32 * (size_t)k + 8);
        M.pos[3 * mp] = x[0];
        M.pos[3 * mp + 1] = x[1];
        M.pos[3 * mp + 2] = x[2];
        M.ver[mp] += 1;
        if (!M.dirty[mp]) geo_full(M, mp);  // (see OP_SET_POSE: no stale clean caches)
        else M.gval[mp] = 0;
      }
      if (tid == 0) res[0] = LM_OK;
      return;
    }
    case OP_UPLOAD: {  // DeviceStore.upload_keyframe devicestore.py:68-78
      if (tid) return;
      M.kf_res[A.a] = 1;
      M.ledger[LG_PERSIST] += (unsigned long long)payload_bytes(M, A.a);
      res[0] = LM_OK;
      return;
    }
    case OP_EVICT: {  // DeviceStore.evict_keyframe devicestore.py:103-109
      if (tid) return;
      M.kf_res[A.a] = 0;
      M.ledger[LG_EVICT] += 1;
      res[0] = LM_OK;
      return;
    }
    case OP_MP_GET: {  // one point's record (refreshing a stale representative descriptor)
      const int mp = A.a;
      if (tid < 32 && M.dirty[mp] && M.alive[mp]) refresh_rep_warp(M, mp, tid);
      __syncthreads();
      PointRec* r = (PointRec*)A.buf;
      int2* o = (int2*)(r + 1);
      const int n = M.nobs[mp];
      for (int k = tid; k < n; k += 1024) o[k] = M.obs[M.ooff[mp] + k];
      if (tid == 0) {
        if (M.dirty[mp] && M.alive[mp]) M.dirty[mp] = 0;  // the dirty list keeps the id; refresh_all skips clean ones
        for (int k = 0; k < 3; ++k) r->pos[k] = M.pos[3 * mp + k];
        r->rep[0] = M.rep[2 * mp];
        r->rep[1] = M.rep[2 * mp + 1];
        r->first_kf = M.first_kf[mp];
        r->alive = M.alive[mp];
        r->found = M.found[mp];
        r->visible = M.visible[mp];
        r->nobs = n;
        for (int l = 0; l < LMAX; ++l) r->counts[l] = l < M.L ? M.counts[(size_t)mp * M.L + l] : 0;
        res[0] = LM_OK;
      }
      return;
    }
    case OP_BOUND: {  // bound_points_of mapmodel.py:291-300: live bound ids in keypoint order
      const int P = bound_points<1024>(M, A.a, sh);
      int* out = (int*)A.buf;
      for (int k = tid; k < P; k += 1024) out[k] = M.s.pts[k];
      if (tid == 0) {
        res[0] = LM_OK;
        res[1] = P;
      }
      return;
    }
    case OP_IMPORT_POINTS: {  // lm_import_snapshot: points 0..n-1, no observations yet
      const int n = A.n;
      // n x 96 B: pos @0 (24), rep @32 (32), first kf @64, found @72, visible @76, alive @80
      const char* b = (const char*)A.buf;
      for (int id = tid; id < n; id += 1024) {
        const char* e = b + 96 * (size_t)id;
        const double* x = (const double*)e;
        for (int k = 0; k < 3; ++k) M.pos[3 * id + k] = x[k];
        M.rep[2 * id] = *(const uint4*)(e + 32);
        M.rep[2 * id + 1] = *(const uint4*)(e + 48);
        M.first_kf[id] = *(const long long*)(e + 64);
        M.found[id] = *(const int*)(e + 72);
        M.visible[id] = *(const int*)(e + 76);
        M.alive[id] = *(const unsigned char*)(e + 80);
        M.nobs[id] = 0;
        M.ocap[id] = 0;
        M.ooff[id] = 0;
        M.gval[id] = 0;
        M.dirty[id] = 0;
      }
      if (tid == 0) {
        M.scal[SC_NEXT_ID] = n;
        res[0] = LM_OK;
      }
      return;
    }
    case OP_GEO_ALL: {  // view-geometry caches of every live clean point (after an import)
      const int n = M.scal[SC_NEXT_ID];
      for (int mp = tid; mp < n; mp += 1024)
        if (M.alive[mp] && !M.dirty[mp] && M.nobs[mp]) geo_full(M, mp);
      if (tid == 0) res[0] = LM_OK;
      return;
    }
    case OP_CORRUPT: {  // fault injection for the audit tests (test_mapmodel.py:238-255)
      if (tid) return;
      if (A.n == 0) M.counts[(size_t)A.a * M.L + A.b] += A.c;
      else covis_global(M, A.a, A.b, A.c);
      res[0] = LM_OK;
      return;
    }
    case OP_LEDGER_ADD: {  // explicit record_neighbor_access / record_small_transfer (devicestore.py:80-101)
      if (tid) return;
      M.ledger[LG_NAIVE] += (unsigned long long)A.v0;
      if (A.n) {  // one small-transfer event of A.v1 bytes (stage: A.b = 1 triangulation, else fusion)
        const unsigned long long ev = M.ledger[LG_SMALL_EVENTS];
        if (ev < (unsigned long long)LG_LOG_CAP) M.lg_log[ev] = A.b ? -(long long)A.v1 - 1 : A.v1;
        M.ledger[LG_SMALL_EVENTS] = ev + 1;
        M.ledger[A.b ? LG_SMALL_TRI : LG_SMALL_FUSE] += (unsigned long long)A.v1;
        M.ledger[LG_NAIVE] += (unsigned long long)A.v1;
        M.ledger[LG_PERSIST] += (unsigned long long)A.v1;
      }
      res[0] = LM_OK;
      return;
    }
    default:
      if (tid == 0) res[0] = LM_ERR_INVALID_ARGUMENT;
  }
}

static int run_op(lm_ctx* ctx, HostMap* m, int map, OpArgs& a, int* res_host, int nres) {
  a.n_slots = m->n_slots;
  const size_t dyn = 13 * (size_t)m->d.kf_cap + 16;  // ranked slots (12 B/slot) + target flags
  k_op<<<1, 1024, dyn, ctx->stream>>>(ctx->d_maps, map, a, m->d_result);
  CHECK_LAUNCH();
  ctx->launches += 1;
  CU(cudaMemcpyAsync(res_host, m->d_result, sizeof(int) * nres, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return LM_OK;
}

static int io_reserve(lm_ctx* ctx, HostMap* m, size_t bytes) {
  if (bytes <= m->io_bytes) return LM_OK;
  CU(cudaStreamSynchronize(ctx->stream));
  if (m->d_io) CU(cudaFree(m->d_io));
  size_t sz = m->io_bytes ? m->io_bytes : 65536;
  while (sz < bytes) sz *= 2;
  CU(cudaMalloc(&m->d_io, sz));
  m->io_bytes = sz;
  return LM_OK;
}

// fire-and-forget op (its status is validated on the host): no result readback, no sync
static int run_op_async(lm_ctx* ctx, HostMap* m, int map, OpArgs& a) {
  a.n_slots = m->n_slots;
  const size_t dyn = 13 * (size_t)m->d.kf_cap + 16;
  k_op<<<1, 1024, dyn, ctx->stream>>>(ctx->d_maps, map, a, m->d_result);
  CHECK_LAUNCH();
  ctx->launches += 1;
  return LM_OK;
}

static int op_status(lm_ctx* ctx, int code, const char* what) {
  switch (code) {
    case LM_OK: return LM_OK;
    case LM_ERR_INVALID_ARGUMENT: return fail(ctx, code, "%s: invalid argument", what);
    case LM_ERR_INVALID_STATE: return fail(ctx, code, "%s: entity is dead", what);
    case LM_ERR_SLOT_CONFLICT: return fail(ctx, code, "%s: slot already bound", what);
    case LM_ERR_CAPACITY: return fail(ctx, code, "%s: device arena capacity exceeded", what);
    default: return fail(ctx, code, "%s: error %d", what, code);
  }
}

// ------------------------------------------------------------------- ABI
// step-kernel launch: programmatic dependent launch  and an optional
// cluster dimension
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(lm_ctx* ctx, void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, int cluster,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (ctx->pdl_now) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 0) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

extern "C" {

static int refresh(lm_ctx* ctx, HostMap* m, int map);
__global__ void __launch_bounds__(256) k_fuse_visible_end(DevMap* maps, const StepArgs* args, lm_step_stats** totals);

int lm_version(void) { return 1; }

int lm_ctx_create(int32_t device, lm_ctx** out) {
  if (!out) return LM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  lm_ctx* ctx = new lm_ctx();
  ctx->device = device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev) {
    *out = ctx;
    return fail(ctx, LM_ERR_CUDA, "no CUDA device %d (%s)", device, cudaGetErrorString(e));
  }
  CU(cudaSetDevice(device));
  CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->stage_stream, cudaStreamNonBlocking));
  CU(cudaMallocHost(&ctx->h_args, sizeof(StepArgs) * kRing * kMaxBatch));
  CU(cudaMalloc(&ctx->d_args, sizeof(StepArgs) * kRing * kMaxBatch));
  CU(cudaMallocHost(&ctx->h_stats, sizeof(lm_step_stats) * kMaxBatch));
  for (int i = 0; i < kRing; ++i) {
    CU(cudaEventCreateWithFlags(&ctx->args_ev[i], cudaEventDisableTiming));
    ctx->args_used[i] = false;
  }
  for (int i = 0; i < kStageRing; ++i) {
    CU(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
    ctx->stage_used[i] = false;
    ctx->h_stage[i] = nullptr;
    ctx->d_stage[i] = nullptr;
  }
  CU(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  CU(cudaFuncSetAttribute(k_fuse_targets, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  // (k_cull / k_fuse_apply / k_fuse_rev: <false> for every launch, <true> for the profile pass)
  CU(cudaFuncSetAttribute(k_fuse_rev<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  CU(cudaFuncSetAttribute(k_fuse_rev<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  CU(cudaFuncSetAttribute(k_op, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  CU(cudaFuncSetAttribute(k_fuse_apply<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_fuse_apply<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_fuse_rev<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_fuse_rev<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_cull<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CULL_DYN_SMEM));
  CU(cudaFuncSetAttribute(k_cull<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_cull<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CU(cudaFuncSetAttribute(k_cull<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CULL_DYN_SMEM));
  CU(cudaFuncSetAttribute(k_tri, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  if (const char* e = getenv("LM_CARVEOUT")) {  // (experiments) shared-memory carve-out hint, percent
    const int pc = atoi(e);
    const void* ks[] = {(const void*)k_insert, (const void*)k_cull<false>, (const void*)k_cull<true>, (const void*)k_select, (const void*)k_prep,
                        (const void*)k_match, (const void*)k_tri, (const void*)k_commit, (const void*)k_fuse_targets,
                        (const void*)k_fuse_geo, (const void*)k_fuse_gather, (const void*)k_fuse_apply<false>, (const void*)k_fuse_apply<true>,
                        (const void*)k_fuse_refresh, (const void*)k_fuse_spec<true>, (const void*)k_fuse_spec<false>,
                        (const void*)k_fuse_spec_pts, (const void*)k_fuse_spec_hit, (const void*)k_fuse_post,
                        (const void*)k_fuse_rev<false>, (const void*)k_fuse_rev<true>, (const void*)k_fuse_visible_end};
    for (const void* k : ks) CU(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
  }
  if (const char* e = getenv("LM_PDL")) ctx->pdl = atoi(e) != 0 ? 1 : 0;
  if (const char* e = getenv("LM_REV_CLUSTER")) ctx->rev_cluster = atoi(e) > 0 ? atoi(e) : 1;
  if (const char* e = getenv("LM_REFRESH_BLOCKS")) ctx->refresh_blocks = atoi(e) > 0 ? atoi(e) : 148;
  if (const char* e = getenv("LM_POST_BLOCKS"))
    ctx->post_blocks = atoi(e) > 0 ? (atoi(e) < POST_BLOCKS ? atoi(e) : POST_BLOCKS) : 148;
  if (const char* e = getenv("LM_REV_WIDE")) {
    int d = 1, o = 1;
    if (sscanf(e, "%d,%d", &d, &o) >= 1) ctx->rev_wide = (d < 1 ? 1 : d > 255 ? 255 : d) | (o < 1 ? 1 : o > 255 ? 255 : o) << 8;
  }
  if (const char* e = getenv("LM_TRI_SLICES")) ctx->tri_slices = atoi(e) > 0 ? (atoi(e) < 32 ? atoi(e) : 32) : 1;
  if (const char* e = getenv("LM_CULL_CLUSTER")) {
    const int v = atoi(e);
    ctx->cull_cluster = v < 1 ? 1 : (v > 16 ? 16 : v);
  }
  if (const char* e = getenv("LM_APPLY_CLUSTER")) {
    const int v = atoi(e);
    ctx->apply_cluster = v < 1 ? 1 : (v > 16 ? 16 : v);
  }
  *out = ctx;
  return LM_OK;
}

int lm_ctx_destroy(lm_ctx* ctx) {
  if (!ctx) return LM_OK;
  if (ctx->stage_stream) cudaStreamSynchronize(ctx->stage_stream);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (HostMap* m : ctx->maps) {
    if (!m) continue;
    for (void* p : m->allocs) cudaFree(p);
    if (m->d_io) cudaFree(m->d_io);
    delete m;
  }
  if (ctx->d_maps) cudaFree(ctx->d_maps);
  if (ctx->d_totals) cudaFree(ctx->d_totals);
  if (ctx->flush_buf) cudaFree(ctx->flush_buf);
  if (ctx->t0) cudaEventDestroy(ctx->t0);
  if (ctx->t1) cudaEventDestroy(ctx->t1);
  for (int i = 0; i < kRing; ++i) cudaEventDestroy(ctx->args_ev[i]);
  for (int i = 0; i < kStageRing; ++i) cudaEventDestroy(ctx->stage_ev[i]);
  for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
  for (auto& v : ctx->prof_steps)
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  if (ctx->h_args) cudaFreeHost(ctx->h_args);
  if (ctx->d_args) cudaFree(ctx->d_args);
  if (ctx->h_stats) cudaFreeHost(ctx->h_stats);
  if (ctx->h_io) cudaFreeHost(ctx->h_io);
  for (int i = 0; i < kStageRing; ++i) {
    if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
    if (ctx->d_stage[i]) cudaFree(ctx->d_stage[i]);
  }
  if (ctx->stage_stream) cudaStreamDestroy(ctx->stage_stream);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return LM_OK;
}

const char* lm_last_error(lm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int lm_ctx_set_pdl(lm_ctx* ctx, int32_t mode) {
  if (!ctx) return LM_ERR_INVALID_ARGUMENT;
  ctx->pdl = mode < 0 ? -1 : (mode ? 1 : 0);
  return LM_OK;
}

int lm_synchronize(lm_ctx* ctx) {
  if (!ctx) return LM_ERR_INVALID_ARGUMENT;
  CU(cudaStreamSynchronize(ctx->stream));
  return LM_OK;
}

static double host_pow(double b, int e) { return pow(b, (double)e); }

int lm_map_create(lm_ctx* ctx, const lm_map_caps* c, int32_t* map_out) {
  if (!ctx || !c || !map_out) return LM_ERR_INVALID_ARGUMENT;
  if (c->num_levels < 1 || c->num_levels > LMAX || !(c->scale_factor > 1.0) || c->max_keyframes < 2 ||
      c->max_keypoints_per_kf < 1 || c->max_keypoints < c->max_keypoints_per_kf || c->max_points < 1 ||
      c->obs_pool_entries < 8)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "invalid map capacities");
  // k_select / k_fuse_targets / k_op stage 12 bytes per keyframe slot in shared memory and
  // the pair-reservation hash packs slot ids into 16 bits
  if (c->max_keyframes > LM_MAX_KF_SLOTS)
    return fail(ctx, LM_ERR_CAPACITY, "max_keyframes %d exceeds the device limit %d", c->max_keyframes,
                LM_MAX_KF_SLOTS);
  // the fusion apply packs keypoint and point ids into 28 bits (reservation key sets)
  if (c->max_keypoints >= (1 << 28) || c->max_points >= (1 << 28))
    return fail(ctx, LM_ERR_CAPACITY, "max_keypoints / max_points must be below 2^28 per map");
  CU(cudaSetDevice(ctx->device));
  HostMap* m = new HostMap();
  m->caps = *c;
  DevMap& d = m->d;
  d.kf_cap = c->max_keyframes;
  d.kp_cap = c->max_keypoints;
  d.kpkf_max = c->max_keypoints_per_kf;
  d.mp_cap = c->max_points;
  d.obs_cap = c->obs_pool_entries;
  d.L = c->num_levels;
  d.min_w = c->min_covis_weight < 1 ? 1 : c->min_covis_weight;
  d.min_obs_keep = c->min_obs_keep;
  d.recent_cap = c->max_points;
  d.kp_rec_bytes = c->keypoint_record_bytes;
  d.desc_bytes = c->descriptor_bytes;
  d.mp_rec_bytes = c->map_point_record_bytes;
  d.sf = c->scale_factor;
  d.log_sf = log(c->scale_factor);
  for (int l = 0; l < LMAX; ++l) {
    d.S[l] = host_pow(c->scale_factor, l);
    d.S2[l] = host_pow(c->scale_factor, 2 * l);
  }
  const size_t K = d.kf_cap, KP = d.kp_cap, MP = d.mp_cap, NK = (size_t)NMAX * d.kpkf_max;
  int rc = LM_OK;
#define A(ptr, n) \
  if ((rc = arena(ctx, m, &(ptr), (n))) != LM_OK) return rc
  A(d.kf_id, K); A(d.kf_state, K); A(d.kf_res, K); A(d.kp_off, K); A(d.kp_n, K);
  A(d.q, 4 * K); A(d.R, 9 * K); A(d.t, 3 * K); A(d.C, 3 * K); A(d.P, 12 * K); A(d.cam, 6 * K);
  A(d.g_cs, K); A(d.g_nx, K); A(d.g_ny, K);
  A(d.cell_start, K * (GRID_CELLS + 1)); A(d.cell_items, KP);
  A(d.ku, KP); A(d.kv, KP); A(d.klev, KP); A(d.kdesc, 2 * KP); A(d.kbind, KP);
  A(d.pos, 3 * MP); A(d.rep, 2 * MP); A(d.alive, MP); A(d.found, MP); A(d.visible, MP); A(d.first_kf, MP);
  A(d.nobs, MP); A(d.ocap, MP); A(d.ooff, MP); A(d.obs, (size_t)d.obs_cap); A(d.counts, MP * d.L);
  A(d.dirty, MP); A(d.dirty_list, MP); A(d.res_pt, MP); A(d.res_slot, KP);
  A(d.res_ex, MP); A(d.res_pair, RES_PAIR); A(d.grp_head, MP);
  A(d.gacc, 3 * MP); A(d.glo, MP); A(d.ghi, MP); A(d.gval, MP); A(d.ver, MP); A(d.hit, MP); A(d.mrg, MP);
  A(d.sp_tag, MP); A(d.sp_j, MP); A(d.sp_ver0, MP); A(d.sp_nobs0, MP); A(d.sp_hit, MP); A(d.sp_rep, 2 * MP);
  A(d.sp_geo, 5 * MP);
  A(d.covis, K * K);
  A(d.recent_id, MP); A(d.recent_born, MP);
  A(d.scal, SC_N); A(d.ledger, LG_N); A(d.lg_log, LG_LOG_CAP);
  Scratch& s = d.s;
  A(s.nbr, NMAX); A(s.deg, NMAX); A(s.F, 9 * NMAX);
  A(s.cur_sorted, d.kpkf_max); A(s.cur_bucket, LMAX + 1);
  A(s.tiles, 3 * (d.kpkf_max / MATCH_TILE + LMAX + 1)); A(s.n_tiles, 1);
  A(s.nb_n, NMAX); A(s.nb_bucket, NMAX * (LMAX + 1)); A(s.nb_j, NK); A(s.nb_desc, 2 * NK);
  A(s.nb_u, NK); A(s.nb_v, NK); A(s.nb_thr, NK); A(s.pick, NK); A(s.bestj, NK);
  A(s.cand_n, NMAX); A(s.cand_i, NK); A(s.cand_j, NK); A(s.cand_d, NK); A(s.cand_st, NK); A(s.cand_X, 3 * NK);
  A(s.win_rank, d.kpkf_max); A(s.crank, NK); A(s.cmeta, 4); A(s.mask_cur, d.kpkf_max); A(s.mask_nbr, d.kpkf_max);
  A(s.targets, TMAX); A(s.n_targets, 1); A(s.rank_buf, (size_t)TMAX * (3 * K + 1) + (size_t)TMAX * K * 2 + 2);
  s.pts_cap = d.kpkf_max;
  A(s.pts, s.pts_cap); A(s.geo, s.pts_cap);
  s.act_cap = TMAX * d.kpkf_max;
  A(s.acts, (size_t)s.act_cap); A(s.act_flag, (size_t)s.act_cap); A(s.vis_flag, (size_t)s.act_cap);
  A(s.pend, (size_t)s.act_cap); A(s.ready, (size_t)s.act_cap); A(s.merge_a, (size_t)s.act_cap); A(s.merge_b, (size_t)s.act_cap); A(s.acts2, (size_t)s.act_cap);
  A(s.blk_cnt, (size_t)s.act_cap / 256 + 2); A(s.blk_off, (size_t)s.act_cap / 256 + 2); A(s.fctl, 8);
  A(s.pass_j, d.kpkf_max); A(s.add_list, (size_t)s.act_cap);
  A(s.def, (size_t)s.act_cap); A(s.dnxt, (size_t)s.act_cap); A(s.gbase, MP);
  A(s.pinfo, 3 * TMAX); A(s.hitpass, (size_t)d.kpkf_max * ((TMAX + 31) / 32)); A(s.pj, (size_t)s.act_cap);
  A(s.pass_of, K); A(s.snap, d.kpkf_max); A(s.chg, d.kpkf_max); A(s.rmark, MP); A(s.die, MP);
  A(s.pmp, (size_t)s.act_cap); A(s.pob, (size_t)s.act_cap); A(s.itag, (size_t)s.act_cap); A(s.ilist, (size_t)s.act_cap);
  A(s.cands, (size_t)s.act_cap); A(s.cneed, (size_t)s.act_cap); A(s.hl_cnt, d.kpkf_max); A(s.hl, (size_t)d.kpkf_max * HL); A(s.hreg, MP); A(s.upts, (size_t)s.act_cap); A(s.sp_list, (size_t)s.act_cap); A(s.sp_obs, (size_t)POST_BLOCKS * 8 * (POST_MAXN + 1));
  A(s.abits, (size_t)TMAX * ((d.kpkf_max + 31) / 32));
  A(m->d_stats, 1); A(m->d_totals, 1); A(m->d_result, 4 + 1024 + TMAX);
#undef A
  s.stats = m->d_stats;
  CU(cudaMemsetAsync(d.res_pt, 0xff, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.res_slot, 0xff, sizeof(unsigned long long) * KP, ctx->stream));
  CU(cudaMemsetAsync(d.res_ex, 0xff, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.res_pair, 0xff, sizeof(unsigned long long) * RES_PAIR, ctx->stream));
  CU(cudaMemsetAsync(d.grp_head, 0, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.rmark, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.die, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.itag, 0, sizeof(int) * d.s.act_cap, ctx->stream));
  CU(cudaMemsetAsync(d.mrg, 0, sizeof(int2) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.hreg, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.sp_tag, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.hit, 0xff, sizeof(int2) * MP, ctx->stream));
  CU(cudaMemsetAsync(s.pass_of, 0xff, sizeof(int) * K, ctx->stream));
  CU(cudaMemsetAsync(s.hitpass, 0, sizeof(unsigned) * d.kpkf_max * ((TMAX + 31) / 32), ctx->stream));
  m->state.assign(K, KF_FREE);
  m->res.assign(K, 0);
  m->prebound.assign(K, 0);
  m->kp_n.assign(K, 0);
  m->kp_off.assign(K, 0);
  m->ids.assign(K, 0);
  ctx->maps.push_back(m);
  *map_out = (int32_t)ctx->maps.size() - 1;
  return upload_maps(ctx);
}

int lm_map_destroy(lm_ctx* ctx, int32_t map) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  CU(cudaStreamSynchronize(ctx->stream));
  for (void* p : m->allocs) CU(cudaFree(p));
  if (m->d_io) CU(cudaFree(m->d_io));
  delete m;
  ctx->maps[map] = nullptr;  // the index is not reused; other maps keep theirs
  return LM_OK;
}

int lm_map_reset(lm_ctx* ctx, int32_t map) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  DevMap& d = m->d;
  const size_t K = d.kf_cap, MP = d.mp_cap;
  CU(cudaMemsetAsync(d.kf_state, 0, sizeof(int) * K, ctx->stream));
  CU(cudaMemsetAsync(d.kf_res, 0, K, ctx->stream));
  CU(cudaMemsetAsync(d.covis, 0, sizeof(int) * K * K, ctx->stream));
  CU(cudaMemsetAsync(d.alive, 0, MP, ctx->stream));
  CU(cudaMemsetAsync(d.nobs, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.ocap, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.counts, 0, sizeof(int) * MP * d.L, ctx->stream));
  CU(cudaMemsetAsync(d.dirty, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.gval, 0, MP, ctx->stream));
  CU(cudaMemsetAsync(d.hit, 0xff, sizeof(int2) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.ver, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.scal, 0, sizeof(int) * SC_N, ctx->stream));
  CU(cudaMemsetAsync(d.ledger, 0, sizeof(unsigned long long) * LG_N, ctx->stream));
  CU(cudaMemsetAsync(m->d_totals, 0, sizeof(lm_step_stats), ctx->stream));
  CU(cudaMemsetAsync(d.res_pt, 0xff, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.res_slot, 0xff, sizeof(unsigned long long) * d.kp_cap, ctx->stream));
  CU(cudaMemsetAsync(d.res_ex, 0xff, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.res_pair, 0xff, sizeof(unsigned long long) * RES_PAIR, ctx->stream));
  CU(cudaMemsetAsync(d.grp_head, 0, sizeof(unsigned long long) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.rmark, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.die, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.itag, 0, sizeof(int) * d.s.act_cap, ctx->stream));
  CU(cudaMemsetAsync(d.mrg, 0, sizeof(int2) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.s.hreg, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaMemsetAsync(d.sp_tag, 0, sizeof(int) * MP, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  m->slot_of.clear();
  std::fill(m->state.begin(), m->state.end(), KF_FREE);
  std::fill(m->res.begin(), m->res.end(), 0);
  m->n_slots = m->kp_head = m->resident = 0;
  return LM_OK;
}

int lm_map_sizes_get(lm_ctx* ctx, int32_t map, lm_map_sizes* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int sc[SC_N];
  CU(cudaMemcpyAsync(sc, m->d.scal, sizeof sc, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  out->n_kf_slots = m->n_slots;
  out->n_points = sc[SC_NEXT_ID];
  out->n_keypoints = m->kp_head;
  out->obs_used = sc[SC_OBS_HEAD];
  out->recent_n = sc[SC_RECENT_N];
  return LM_OK;
}

int lm_kf_stage(lm_ctx* ctx, int32_t map, int64_t kf_id, const double quat[4], const double trans[3],
                const double cam[6], int32_t n, const double* u, const double* v, const int64_t* level,
                const uint8_t* desc, const int64_t* bindings) {
  HostMap* m;
  int rc = check_map(ctx, map, &m, false);  // (staging is ordered on its own stream)
  if (rc) return rc;
  DevMap& d = m->d;
  if (m->slot_of.count(kf_id)) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "duplicate keyframe id %lld", (long long)kf_id);
  if (n < 0 || n > d.kpkf_max)
    return fail(ctx, LM_ERR_CAPACITY, "keyframe has %d keypoints, map limit %d", n, d.kpkf_max);
  if (m->n_slots >= d.kf_cap) return fail(ctx, LM_ERR_CAPACITY, "keyframe slots exhausted (%d)", d.kf_cap);
  if (m->kp_head + n > d.kp_cap) return fail(ctx, LM_ERR_CAPACITY, "keypoint pool exhausted (%d)", d.kp_cap);
  if (!(cam[0] > 0 && cam[1] > 0 && cam[4] > 0 && cam[5] > 0))
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "bad intrinsics");
  for (int i = 0; i < n; ++i)
    if (level[i] < 0 || level[i] >= d.L) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "keypoint level outside pyramid");
  // staging buffer (ring)
  const size_t need = sizeof(StageHdr) + (size_t)n * (8 + 8 + 32 + 4 + 1) + 64;
  const long long sidx = ctx->stage_pos++;
  const int b = (int)(sidx % kStageRing);
  if (ctx->stage_used[b]) CU(cudaEventSynchronize(ctx->stage_ev[b]));
  if (ctx->stage_bytes < need) {
    const size_t sz = need < ((size_t)d.kpkf_max * 53 + sizeof(StageHdr) + 64) ? ((size_t)d.kpkf_max * 53 + sizeof(StageHdr) + 64) : need;
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaStreamSynchronize(ctx->stage_stream));
    for (int i = 0; i < kStageRing; ++i) {
      if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
      if (ctx->d_stage[i]) cudaFree(ctx->d_stage[i]);
      CU(cudaMallocHost(&ctx->h_stage[i], sz));
      CU(cudaMalloc(&ctx->d_stage[i], sz));
      ctx->stage_used[i] = false;
    }
    ctx->stage_bytes = sz;
  }
  unsigned char* hb = ctx->h_stage[b];
  StageHdr* h = (StageHdr*)hb;
  const int slot = m->n_slots;
  h->slot = slot;
  h->n = n;
  h->kp_off = m->kp_head;
  h->kf_id = kf_id;
  for (int k = 0; k < 4; ++k) h->q[k] = quat[k];
  for (int k = 0; k < 3; ++k) h->t[k] = trans[k];
  for (int k = 0; k < 6; ++k) h->cam[k] = cam[k];
  quat_to_rot(h->q, h->R);
  camera_center(h->R, h->t, h->C);
  proj_matrix(cam[0], cam[1], cam[2], cam[3], h->R, h->t, h->P);
  const double big = cam[4] > cam[5] ? cam[4] : cam[5];
  double cs = 16.0;
  while (ceil(cam[4] / cs) * ceil(cam[5] / cs) > GRID_CELLS) cs *= 2.0;
  (void)big;
  h->cs = cs;
  h->nx = (int)ceil(cam[4] / cs);
  h->ny = (int)ceil(cam[5] / cs);
  double* pu = (double*)(hb + sizeof(StageHdr));
  double* pv = pu + n;
  unsigned char* pd = (unsigned char*)(pv + n);
  int* pb = (int*)(pd + 32 * (size_t)n);
  unsigned char* pl = (unsigned char*)(pb + n);
  memcpy(pu, u, sizeof(double) * n);
  memcpy(pv, v, sizeof(double) * n);
  memcpy(pd, desc, 32 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    pb[i] = bindings ? (int)bindings[i] : -1;
    pl[i] = (unsigned char)level[i];
  }
  CU(cudaMemcpyAsync(ctx->d_stage[b], hb, need, cudaMemcpyHostToDevice, ctx->stage_stream));
  k_stage<<<1, 1024, 0, ctx->stage_stream>>>(d, ctx->d_stage[b]);
  CHECK_LAUNCH();
  ctx->launches += 1;
  CU(cudaEventRecord(ctx->stage_ev[b], ctx->stage_stream));
  ctx->stage_used[b] = true;
  ctx->last_stage_b = b;
  ctx->stage_unjoined = true;
  m->slot_of[kf_id] = slot;
  m->state[slot] = KF_STAGED;
  m->prebound[slot] = bindings != nullptr;
  m->kp_n[slot] = n;
  m->kp_off[slot] = m->kp_head;
  m->ids[slot] = kf_id;
  m->n_slots++;
  m->kp_head += n;
  return LM_OK;
}

// ------------------------------------------------------------------- steps

// per-step statistics into the running totals, field-parallel: thread k adds summed field k
// (a table of offsets), so every load is independent and nothing spills (a single thread
// copying both records whole needed 255 registers + 600 B of spills: ~10 us per step)
#define LM_SUM32(f) {(int)offsetof(lm_step_stats, f), 4}
#define LM_SUM64(f) {(int)offsetof(lm_step_stats, f), 8}
struct SumField {
  int off, size;
};
__constant__ SumField k_sum_fields[] = {
    LM_SUM32(created), LM_SUM32(conflicts), LM_SUM32(degenerate), LM_SUM32(gate_parallax), LM_SUM32(gate_depth),
    LM_SUM32(gate_reprojection), LM_SUM32(gate_scale), LM_SUM32(n_neighbors), LM_SUM32(n_targets),
    LM_SUM32(merged), LM_SUM32(observations_added), LM_SUM32(stale), LM_SUM32(culled), LM_SUM32(n_candidates),
    LM_SUM64(match_pairs), LM_SUM64(fuse_bytes), LM_SUM64(fuse_passes), LM_SUM64(fuse_points),
    LM_SUM64(fuse_actions), LM_SUM64(apply_rounds), LM_SUM64(rev_passes_acting), LM_SUM64(rev_passes_redo),
    LM_SUM64(fuse_bytes_rev), LM_SUM64(rev_mergeable),
#define LM_ARR(f, k) {(int)(offsetof(lm_step_stats, f) + 8 * (k)), 8}
    LM_ARR(fuse_cycles, 0), LM_ARR(fuse_cycles, 1), LM_ARR(fuse_cycles, 2), LM_ARR(fuse_cycles, 3),
    LM_ARR(fuse_cycles, 4), LM_ARR(fuse_cycles, 5), LM_ARR(fuse_cycles, 6), LM_ARR(fuse_cycles, 7),
    LM_ARR(fuse_cycles, 8), LM_ARR(fuse_cycles, 9), LM_ARR(fuse_cycles, 10), LM_ARR(fuse_cycles, 11),
    LM_ARR(fuse_cycles, 12), LM_ARR(fuse_cycles, 13), LM_ARR(fuse_cycles, 14), LM_ARR(fuse_cycles, 15),
    LM_ARR(dbg, 0), LM_ARR(dbg, 1), LM_ARR(dbg, 2), LM_ARR(dbg, 3), LM_ARR(dbg, 4), LM_ARR(dbg, 5),
    LM_ARR(dbg, 6), LM_ARR(dbg, 7), LM_ARR(dbg, 8), LM_ARR(dbg, 9), LM_ARR(dbg, 10), LM_ARR(dbg, 11),
    LM_ARR(dbg, 12), LM_ARR(dbg, 13), LM_ARR(dbg, 14), LM_ARR(dbg, 15),
    LM_ARR(borderline, 0), LM_ARR(borderline, 1), LM_ARR(borderline, 2), LM_ARR(borderline, 3),
    LM_SUM64(match_second_half),
#undef LM_ARR
};
#undef LM_SUM32
#undef LM_SUM64
constexpr int kSumFields = sizeof(k_sum_fields) / sizeof(SumField);

// the step's statistics into the map's running totals (threads 0..kSumFields of one block)
__device__ __forceinline__ void end_step(const DevMap& M, lm_step_stats* totals) {
  char* st = (char*)M.s.stats;
  char* t = (char*)totals;
  const int k = threadIdx.x;
  if (k < kSumFields) {
    const SumField f = k_sum_fields[k];
    if (f.size == 4) *(int*)(t + f.off) += *(const int*)(st + f.off);
    else *(long long*)(t + f.off) += *(const long long*)(st + f.off);
  } else if (k == kSumFields) {
    const int err = M.scal[SC_ERR], soft = M.scal[SC_SOFT];
    const int e = err ? err : soft;
    ((lm_step_stats*)st)->error = e;
    ((lm_step_stats*)t)->error = err;
    ((lm_step_stats*)t)->first_new_id += 1;  // steps accumulated
  }
}

// last kernel of a step: the reverse passes' deferred visible counters (thread per item),
// then the last block of each map to finish adds the step's statistics to the running totals
// (one launch fewer than a separate end kernel)
__global__ void __launch_bounds__(256) k_fuse_visible_end(DevMap* maps, const StepArgs* args,
                                                          lm_step_stats** totals) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  visible_item(M, A);
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&M.s.fctl[FC_DONE], 1) == (int)(gridDim.x * gridDim.y) - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  end_step(M, totals[A.map]);
  if (threadIdx.x == 0) M.s.fctl[FC_DONE] = 0;
}

static int launch_steps(lm_ctx* ctx, int n, const int32_t* maps, StepArgs* args) {
  if (n < 1 || n > kMaxBatch) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "batch of %d maps", n);
  const int e = ctx->ring_pos++ % kRing;
  if (ctx->args_used[e]) CU(cudaEventSynchronize(ctx->args_ev[e]));
  StepArgs* h = ctx->h_args + (size_t)e * kMaxBatch;
  StepArgs* dv = ctx->d_args + (size_t)e * kMaxBatch;
  int tiles = 1, slots = 1, kfcap = 2, nbr_dim = 1, kpkf = 1, tfuse = 1;
  bool any_cull = false, any_create = false, any_fuse = false;
  for (int k = 0; k < n; ++k) {
    HostMap* m = ctx->maps[maps[k]];
    any_cull |= args[k].do_cull != 0;
    any_create |= args[k].do_create != 0;
    any_fuse |= args[k].do_fuse != 0;
    h[k] = args[k];
    h[k].map = maps[k];
    const int want = args[k].explicit_nbr ? 1 : (args[k].n_nbr_req < NMAX ? args[k].n_nbr_req : NMAX);
    nbr_dim = want > nbr_dim ? want : nbr_dim;
    kpkf = m->d.kpkf_max > kpkf ? m->d.kpkf_max : kpkf;
    if (args[k].do_fuse) {
      const int tf = args[k].fc.n1 + args[k].fc.n1 * args[k].fc.n2;
      tfuse = tf > tfuse ? (tf < TMAX ? tf : TMAX) : tfuse;
    }
    const int t = m->d.kpkf_max / MATCH_TILE + m->d.L + 1;
    tiles = t > tiles ? t : tiles;
    slots = m->n_slots > slots ? m->n_slots : slots;
    kfcap = m->d.kf_cap > kfcap ? m->d.kf_cap : kfcap;
  }
  DevMap* dmaps = ctx->d_maps;
  // reverse passes target the current keyframe; staging it in shared memory (LM_REV_SMEM=1)
  // measured slower on B200: the carve-out it needs shrinks the L1 that the kernel's
  // point/observation loads live in (C2: 45.3 -> 43.1 ms per 200 keyframes without it)
  static const bool rev_stage = getenv("LM_REV_SMEM") != nullptr;
  size_t rev_smem = (size_t)kpkf * (16 + 1 + 32 + 4) + 4 * (GRID_CELLS + 1) + 256;
  if (rev_smem > 160 * 1024 || !rev_stage) rev_smem = 0;
  CU(cudaMemcpyAsync(dv, h, sizeof(StepArgs) * n, cudaMemcpyHostToDevice, ctx->stream));
  const size_t dyn = 12 * (size_t)kfcap;
  std::vector<cudaEvent_t> evs;
  auto mark = [&]() -> int {
    if (!ctx->prof) return LM_OK;
    cudaEvent_t ev;
    if (ctx->prof_pool.empty()) {
      CU(cudaEventCreate(&ev));
    } else {
      ev = ctx->prof_pool.back();
      ctx->prof_pool.pop_back();
    }
    CU(cudaEventRecord(ev, ctx->stream));
    evs.push_back(ev);
    return LM_OK;
  };
  int rc = LM_OK;
  const bool pdl = ctx->pdl < 0 ? n == 1 : ctx->pdl == 1;
  ctx->pdl_now = pdl;
  // a stage no entry of the batch runs is not launched (its kernels would only return): the
  // single-stage calls of the reference-shaped API (cull, create_map_points, run_fusion) pay
  // for their own stage only. The profiled pass launches everything (fixed event layout).
  if (ctx->prof) any_cull = any_create = any_fuse = true;
  int launched = 2;  // k_insert (zeroes the step's statistics) and k_fuse_visible_end (folds them)
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_insert, dim3(n), dim3(256), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  if (any_cull) {
    // recent-point cull: one cluster per map, as wide as the batch leaves SMs for
    int cl = ctx->cull_cluster / n;
    cl = cl < 1 ? 1 : cl;
    CU(launch_k(ctx, ctx->prof ? k_cull<true> : k_cull<false>, dim3(n * cl), dim3(1024), CULL_DYN_SMEM, cl, dmaps,
                (const StepArgs*)dv));
    launched += 1;
  }
  if ((rc = mark())) return rc;
  if (any_create) {
  // k_select and k_fuse_targets run their first part before waiting for their predecessor,
  // which is safe only behind the kernel they were written against (k_cull, k_commit_write):
  // behind any other predecessor they are launched without the PDL attribute (full order)
  ctx->pdl_now = pdl && any_cull;
  CU(launch_k(ctx, k_select, dim3(n), dim3(256), dyn, 0, dmaps, dv, slots));
  ctx->pdl_now = pdl;
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_prep, dim3(1 + nbr_dim, n), dim3(256), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_match, dim3(nbr_dim, tiles, n), dim3(MATCH_WARPS * 32), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  {
    // triangulation slices per neighbour (LM_TRI_SLICES), each with the compacted survivors
    // in shared memory; one slice reading them from global memory past 96 KB
    const size_t tsm = 8 * (size_t)kpkf;
    const int sl = tsm <= 96 * 1024 ? ctx->tri_slices : 1;
    CU(launch_k(ctx, k_tri, dim3(nbr_dim, sl, n), dim3(256), sl > 1 ? tsm : 0, 0, dmaps, dv));
  }
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_commit, dim3(n), dim3(1024), 0, 0, dmaps, dv));
  CU(launch_k(ctx, k_commit_write, dim3((kpkf + 127) / 128, NMAX, n), dim3(128), 0, 0, dmaps, dv));
  launched += 6;
  }  // any_create
  if ((rc = mark())) return rc;
  if (any_fuse) {
  ctx->pdl_now = pdl && any_create;
  CU(launch_k(ctx, k_fuse_targets, dim3(n), dim3(1024), dyn + kfcap + 16, 0, dmaps, dv, slots));
  ctx->pdl_now = pdl;
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_fuse_geo, dim3((kpkf + 7) / 8, n), dim3(256), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_fuse_gather, dim3((tfuse * kpkf + 255) / 256, n), dim3(256), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  {
    // forward apply: one cluster per map, as wide as the batch leaves SMs for
    int cl = ctx->apply_cluster / n;
    cl = cl < 1 ? 1 : (cl > ctx->apply_cluster ? ctx->apply_cluster : cl);
    CU(launch_k(ctx, ctx->prof ? k_fuse_apply<true> : k_fuse_apply<false>, dim3(n * cl), dim3(APPLY_THREADS), 0, cl,
                dmaps, (const StepArgs*)dv));
  }
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_fuse_refresh, dim3(ctx->refresh_blocks, n), dim3(256), 0, 0, dmaps, dv));
  if ((rc = mark())) return rc;
  if (n == 1) {
    CU(launch_k(ctx, k_fuse_spec<true>, dim3((kpkf + 255) / 256, tfuse, n), dim3(256), 0, 0, dmaps, dv));
  } else {  // batches: one gather per distinct point instead of one per (pass, point)
    CU(launch_k(ctx, k_fuse_spec_pts, dim3((kpkf + 255) / 256, tfuse, n), dim3(256), 0, 0, dmaps, dv));
    CU(launch_k(ctx, k_fuse_spec_hit, dim3(16, n), dim3(256), 0, 0, dmaps, dv));
    CU(launch_k(ctx, k_fuse_spec<false>, dim3((kpkf + 255) / 256, tfuse, n), dim3(256), 0, 0, dmaps, dv));
    launched += 2;
  }
  if ((rc = mark())) return rc;
  CU(launch_k(ctx, k_fuse_post, dim3(ctx->post_blocks, n), dim3(256), 0, 0, dmaps, dv));
  {
    // reverse walk: one cluster per map, CTA 0 walks, the others help with direct passes
    int cl = ctx->rev_cluster / n;
    cl = cl < 1 ? 1 : cl;
    CU(launch_k(ctx, ctx->prof ? k_fuse_rev<true> : k_fuse_rev<false>, dim3(n * cl), dim3(REV_THREADS), rev_smem, cl,
                dmaps, dv, (int)rev_smem,
                ctx->rev_wide));
  }
  launched += 8;
  }  // any_fuse
  if ((rc = mark())) return rc;
  // (without fusion one block per map: no pass items, the block folds the statistics)
  CU(launch_k(ctx, k_fuse_visible_end, any_fuse ? dim3((kpkf + 255) / 256, tfuse, n) : dim3(1, 1, n), dim3(256), 0, 0,
              dmaps, dv, ctx->d_totals));
  if ((rc = mark())) return rc;
  ctx->launches += launched;
  if (ctx->prof) ctx->prof_steps.push_back(evs);
  CHECK_LAUNCH();
  CU(cudaEventRecord(ctx->args_ev[e], ctx->stream));
  ctx->args_used[e] = true;
  return LM_OK;
}

static int fill_args(lm_ctx* ctx, HostMap* m, int64_t kf_id, const lm_step_params* p, StepArgs& a, bool insert,
                     bool upload = true) {
  int slot;
  int rc = slot_of(ctx, m, kf_id, &slot, false);
  if (rc) return rc;
  memset(&a, 0, sizeof a);
  a.cur = slot;
  a.do_insert = 0;
  if (m->state[slot] == KF_STAGED) {
    if (!insert) return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld is staged, not inserted", (long long)kf_id);
    a.do_insert = 1;
    a.do_upload = upload;
    if (upload && m->resident >= m->caps.store_capacity && m->caps.store_capacity > 0)
      return fail(ctx, LM_ERR_CAPACITY, "store capacity %d exceeded; size the pre-allocation", m->caps.store_capacity);
  } else if (m->state[slot] != KF_LIVE) {
    return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld is dead", (long long)kf_id);
  }
  if (p) {
    a.n_nbr_req = p->neighbor_count;
    a.do_cull = p->do_cull;
    a.do_create = p->do_create;
    a.do_fuse = p->do_fuse;
    a.processed = p->processed_index;
    a.mc = p->match;
    a.gc = p->gate;
    a.fc = p->fuse;
    a.cc = p->cull;
  }
  if (a.n_nbr_req > NMAX) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "neighbor_count > %d", NMAX);
  // the new keyframe's covisibility row is empty unless it was staged with pre-bound slots,
  // so neighbour selection does not depend on the cull (LM_SELECT_EARLY=0 disables)
  static const bool early_ok = getenv("LM_SELECT_EARLY") == nullptr || atoi(getenv("LM_SELECT_EARLY")) != 0;
  a.select_early = early_ok && a.do_create && !a.explicit_nbr && (!a.do_cull || (a.do_insert && !m->prebound[slot]));
  a.prebound = m->prebound[slot];
  if (a.do_fuse && a.fc.n1 + a.fc.n1 * a.fc.n2 > TMAX)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "n1 + n1*n2 > %d", TMAX);
  return LM_OK;
}

static void after_insert(HostMap* m, const StepArgs& a) {
  if (a.do_insert) m->state[a.cur] = KF_LIVE;
  if (a.do_upload && !m->res[a.cur]) {
    m->res[a.cur] = 1;
    m->resident++;
  }
}

static int step_error(lm_ctx* ctx, int code, int map) {
  if (code == LM_ERR_INVALID_STATE)
    return fail(ctx, code, "map %d: a stage accessed a non-resident keyframe (upload it to the store first)", map);
  if (code == LM_ERR_CAPACITY) return fail(ctx, code, "map %d: device arena capacity exceeded", map);
  return fail(ctx, code, "map %d: invalid pre-bound slot or device error %d", map, code);
}

static int run_batch(lm_ctx* ctx, int n, const int32_t* maps, StepArgs* args, lm_step_stats* out) {
  int rc = launch_steps(ctx, n, maps, args);
  if (rc) return rc;
  CHECK_LAUNCH();
  for (int k = 0; k < n; ++k) after_insert(ctx->maps[maps[k]], args[k]);
  if (!out) return LM_OK;
  for (int k = 0; k < n; ++k)
    CU(cudaMemcpyAsync(ctx->h_stats + k, ctx->maps[maps[k]]->d_stats, sizeof(lm_step_stats), cudaMemcpyDeviceToHost,
                       ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  memcpy(out, ctx->h_stats, sizeof(lm_step_stats) * n);
  for (int k = 0; k < n; ++k)
    if (out[k].error) return step_error(ctx, out[k].error, maps[k]);
  return LM_OK;
}

int lm_step(lm_ctx* ctx, int32_t map, int64_t kf_id, const lm_step_params* p, lm_step_stats* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  StepArgs a;
  rc = fill_args(ctx, m, kf_id, p, a, true);
  if (rc) return rc;
  return run_batch(ctx, 1, &map, &a, out);
}

int lm_step_batch(lm_ctx* ctx, int32_t n, const int32_t* maps, const int64_t* kf_ids, const lm_step_params* p,
                  lm_step_stats* out) {
  if (!ctx) return LM_ERR_INVALID_ARGUMENT;
  if (n < 1 || n > kMaxBatch || !maps || !kf_ids || !p)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "batch of %d maps (1..%d, maps/kf_ids/params required)", n, kMaxBatch);
  std::vector<StepArgs> args(n);
  for (int k = 0; k < n; ++k) {
    HostMap* m;
    int rc = check_map(ctx, maps[k], &m);
    if (rc) return rc;
    // every kernel of the batch runs one CTA (cluster) per entry on that entry's map: a
    // map listed twice would be stepped twice concurrently (a data race), so reject it
    for (int q = 0; q < k; ++q)
      if (maps[q] == maps[k]) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "map %d listed twice in one batch", maps[k]);
    rc = fill_args(ctx, m, kf_ids[k], p + k, args[k], true);  // one lm_step_params per entry
    if (rc) return rc;
  }
  return run_batch(ctx, n, maps, args.data(), out);
}

int lm_step_stats_fetch(lm_ctx* ctx, int32_t n, const int32_t* maps, lm_step_stats* out) {
  for (int k = 0; k < n; ++k) {
    HostMap* m;
    int rc = check_map(ctx, maps[k], &m);
    if (rc) return rc;
    CU(cudaMemcpyAsync(out + k, m->d_stats, sizeof(lm_step_stats), cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < n; ++k)  // async steps surface device errors here, like run_batch does
    if (out[k].error) return step_error(ctx, out[k].error, maps[k]);
  return LM_OK;
}

static int single_stage(lm_ctx* ctx, int32_t map, int64_t kf_id, lm_step_params& p, lm_step_stats* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  rc = slot_of(ctx, m, kf_id, &slot, true);
  if (rc) return rc;
  lm_step_stats tmp;
  return lm_step(ctx, map, kf_id, &p, out ? out : &tmp);
}

static_assert(sizeof(lm_kf_record_hdr) == 160, "record header layout");

uint64_t lm_kf_record_bytes(int32_t n, uint32_t flags) {
  if (n < 0) return 0;
  const uint64_t nn = (uint64_t)n;
  return sizeof(lm_kf_record_hdr) + 16 * nn + ((nn + 7) & ~7ull) + 32 * nn + ((flags & LM_REC_BINDINGS) ? 8 * nn : 0);
}

int lm_kf_stage_record(lm_ctx* ctx, int32_t map, const void* record, uint64_t bytes, int64_t* kf_id_out) {
  if (!ctx || !record) return LM_ERR_INVALID_ARGUMENT;
  HostMap* m;
  int rc = check_map(ctx, map, &m, false);
  if (rc) return rc;
  if (bytes < sizeof(lm_kf_record_hdr)) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "record shorter than its header");
  lm_kf_record_hdr h;
  memcpy(&h, record, sizeof h);
  if (h.magic != LM_REC_MAGIC || h.version != LM_REC_VERSION || h.header_bytes != sizeof(lm_kf_record_hdr))
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "not an LMKF v1 keyframe record");
  if ((h.flags & ~LM_REC_BINDINGS) != 0) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown record flags %u", h.flags);
  if (h.n > (uint32_t)0x7fffffff || lm_kf_record_bytes((int32_t)h.n, h.flags) != bytes)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "record size %llu does not match %u keypoints", (unsigned long long)bytes, h.n);
  if (h.num_levels != m->d.L || h.scale_factor != m->d.sf)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "record pyramid (%d levels, %g) differs from the map's (%d, %g)",
                h.num_levels, h.scale_factor, m->d.L, m->d.sf);
  const int n = (int)h.n;
  const unsigned char* p = (const unsigned char*)record + sizeof(lm_kf_record_hdr);
  const double* u = (const double*)p;
  const double* v = u + n;
  const unsigned char* lv8 = (const unsigned char*)(v + n);
  const uint8_t* desc = lv8 + ((n + 7) & ~7);
  const int64_t* bind = (h.flags & LM_REC_BINDINGS) ? (const int64_t*)(desc + 32 * (size_t)n) : nullptr;
  std::vector<int64_t> level(n);
  for (int i = 0; i < n; ++i) level[i] = lv8[i];
  const double cam[6] = {h.fx, h.fy, h.cx, h.cy, (double)h.width, (double)h.height};
  rc = lm_kf_stage(ctx, map, h.kf_id, h.quat, h.trans, cam, n, u, v, level.data(), desc, bind);
  if (rc == LM_OK && kf_id_out) *kf_id_out = h.kf_id;
  return rc;
}

int lm_kf_insert(lm_ctx* ctx, int32_t map, int64_t kf_id) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  rc = slot_of(ctx, m, kf_id, &slot, false);
  if (rc) return rc;
  if (m->state[slot] != KF_STAGED) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "duplicate keyframe id %lld", (long long)kf_id);
  // MapModel.insert_keyframe only: residency and the upload ledger entry are the store's
  // (lm_kf_upload), as in the reference pipeline (pipeline.py:163-164)
  StepArgs a;
  if ((rc = fill_args(ctx, m, kf_id, nullptr, a, true, false))) return rc;
  // without pre-bound slots the insert cannot fail on the device: no readback, no sync
  lm_step_stats st;
  return run_batch(ctx, 1, &map, &a, m->prebound[slot] ? &st : nullptr);
}

int lm_create_map_points(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t neighbor_count, const lm_match_cfg* mc,
                         const lm_gate_cfg* gc, lm_step_stats* out) {
  if (!mc || !gc) return LM_ERR_INVALID_ARGUMENT;
  lm_step_params p;
  memset(&p, 0, sizeof p);
  p.neighbor_count = neighbor_count;
  p.do_create = neighbor_count > 0;
  p.match = *mc;
  p.gate = *gc;
  return single_stage(ctx, map, kf_id, p, out);
}

int lm_run_fusion(lm_ctx* ctx, int32_t map, int64_t kf_id, const lm_fuse_cfg* fc, lm_step_stats* out) {
  if (!fc) return LM_ERR_INVALID_ARGUMENT;
  lm_step_params p;
  memset(&p, 0, sizeof p);
  p.do_fuse = 1;
  p.fuse = *fc;
  return single_stage(ctx, map, kf_id, p, out);
}

int lm_cull_recent(lm_ctx* ctx, int32_t map, int32_t processed_index, const lm_cull_cfg* cc, int32_t* culled) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  // any live keyframe works as the step anchor; the cull stage does not read it
  int anchor = -1;
  for (int s = 0; s < m->n_slots; ++s)
    if (m->state[s] == KF_LIVE) {
      anchor = s;
      break;
    }
  if (anchor < 0) {
    if (culled) *culled = 0;
    return LM_OK;
  }
  lm_step_params p;
  memset(&p, 0, sizeof p);
  p.do_cull = 1;
  p.processed_index = processed_index;
  p.cull = *cc;
  lm_step_stats st;
  rc = lm_step(ctx, map, m->ids[anchor], &p, &st);
  if (culled) *culled = st.culled;
  return rc;
}

// pinned host scratch of at least `bytes` (callers synchronise before returning, so the
// buffer is free at entry)
static int host_io(lm_ctx* ctx, size_t bytes, unsigned char** out) {
  if (bytes > ctx->h_io_bytes) {
    if (ctx->h_io) cudaFreeHost(ctx->h_io);
    ctx->h_io = nullptr;
    ctx->h_io_bytes = 0;
    size_t sz = 1 << 16;
    while (sz < bytes) sz *= 2;
    CU(cudaMallocHost(&ctx->h_io, sz));
    ctx->h_io_bytes = sz;
  }
  *out = ctx->h_io;
  return LM_OK;
}

int lm_cull_recent_list(lm_ctx* ctx, int32_t map, int32_t processed_index, const lm_cull_cfg* cc, int32_t n,
                        const int64_t* ids, const int32_t* born, int64_t* removed, int32_t* n_removed,
                        int64_t* keep_ids, int32_t* keep_born, int32_t* n_keep) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (!cc) return LM_ERR_INVALID_ARGUMENT;
  *n_removed = 0;
  *n_keep = 0;
  if (n <= 0) return lm_recent_import(ctx, map, ids, born, 0);
  if (n > m->d.recent_cap) return fail(ctx, LM_ERR_CAPACITY, "recent list too long");
  int anchor = -1;  // any live keyframe anchors the cull-only step (the stage does not read it)
  for (int s = 0; s < m->n_slots && anchor < 0; ++s)
    if (m->state[s] == KF_LIVE) anchor = s;
  // one round trip: the list in, both alive ranges, the kept list and the step's statistics
  // out, through pinned scratch. An id that names no map point is skipped, as the reference
  // skips an entry whose point it cannot find (culling.py:44-46 `mp is None`): ids outside
  // the point arena are not uploaded; ids not created yet are dead (alive = 0) on the device.
  const size_t N = (size_t)n;
  std::vector<int> kept_in;
  kept_in.reserve(N);
  long long lo = m->d.mp_cap, hi = -1, prev = -1;
  bool increasing = true;
  for (int k = 0; k < n; ++k) {
    if (ids[k] < 0 || ids[k] >= m->d.mp_cap) continue;
    kept_in.push_back(k);
    lo = ids[k] < lo ? ids[k] : lo;
    hi = ids[k] > hi ? ids[k] : hi;
    increasing &= ids[k] > prev;
    prev = ids[k];
  }
  const int nv = (int)kept_in.size();
  if (!increasing) {  // (the pipeline appends ids in creation order; anything else is checked)
    // a point listed twice would be classified twice in one pass (a double kill), where the
    // reference's second visit finds it already dead: rejected instead
    std::vector<long long> sorted;
    sorted.reserve(nv);
    for (int q = 0; q < nv; ++q) sorted.push_back(ids[kept_in[q]]);
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
      return fail(ctx, LM_ERR_INVALID_ARGUMENT, "map point listed twice in the probation list");
  }
  if (nv == 0) return lm_recent_import(ctx, map, ids, born, 0);
  unsigned char* hb;
  const size_t R = (size_t)(hi - lo + 1);
  const size_t o_id = 0, o_born = o_id + 4 * N, o_n = o_born + 4 * N, o_stats = (o_n + 4 + 7) & ~(size_t)7;
  const size_t o_kid = o_stats + sizeof(lm_step_stats), o_kborn = o_kid + 4 * N, o_kn = o_kborn + 4 * N;
  const size_t o_before = o_kn + 4, o_after = o_before + R;
  if ((rc = host_io(ctx, o_after + R, &hb))) return rc;
  int* hid = (int*)(hb + o_id);
  int* hborn = (int*)(hb + o_born);
  for (int q = 0; q < nv; ++q) {
    hid[q] = (int)ids[kept_in[q]];
    hborn[q] = born[kept_in[q]];
  }
  *(int*)(hb + o_n) = nv;
  CU(cudaMemcpyAsync(hb + o_before, m->d.alive + lo, R, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(m->d.recent_id, hb + o_id, 4 * (size_t)nv, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(m->d.recent_born, hb + o_born, 4 * (size_t)nv, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(m->d.scal + SC_RECENT_N, hb + o_n, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  if (anchor >= 0) {
    lm_step_params p;
    memset(&p, 0, sizeof p);
    p.do_cull = 1;
    p.processed_index = processed_index;
    p.cull = *cc;
    StepArgs a;
    if ((rc = fill_args(ctx, m, m->ids[anchor], &p, a, true))) return rc;
    if ((rc = run_batch(ctx, 1, &map, &a, nullptr))) return rc;  // (no readback: the copies below)
    CU(cudaMemcpyAsync(hb + o_stats, m->d_stats, sizeof(lm_step_stats), cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(cudaMemcpyAsync(hb + o_after, m->d.alive + lo, R, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hb + o_kn, m->d.scal + SC_RECENT_N, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hb + o_kid, m->d.recent_id, 4 * (size_t)nv, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hb + o_kborn, m->d.recent_born, 4 * (size_t)nv, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (anchor >= 0) {
    const int err = ((const lm_step_stats*)(hb + o_stats))->error;
    if (err) return step_error(ctx, err, map);
  }
  const unsigned char* before = hb + o_before;
  const unsigned char* after = hb + o_after;
  int r = 0;
  for (int q = 0; q < nv; ++q) {  // removed = alive before, dead after, in probation order
    const long long id = ids[kept_in[q]];
    if (before[id - lo] && !after[id - lo]) removed[r++] = id;
  }
  *n_removed = r;
  const int kn = *(const int*)(hb + o_kn);
  if (kn < 0 || kn > nv) return fail(ctx, LM_ERR_INVALID_STATE, "probation list grew in a cull (%d > %d)", kn, nv);
  const int* kid = (const int*)(hb + o_kid);
  for (int k = 0; k < kn; ++k) keep_ids[k] = kid[k];
  memcpy(keep_born, hb + o_kborn, 4 * (size_t)kn);
  *n_keep = kn;
  return LM_OK;
}

int lm_search(lm_ctx* ctx, int32_t map, int64_t cur_kf, int64_t nbr_kf, const lm_match_cfg* mc,
              const uint8_t* unbound_cur, const uint8_t* unbound_nbr, lm_candidate* out, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int cs, ns;
  if ((rc = slot_of(ctx, m, cur_kf, &cs, false)) || (rc = slot_of(ctx, m, nbr_kf, &ns, false))) return rc;
  if (m->state[cs] == KF_FREE || m->state[ns] == KF_FREE) return fail(ctx, LM_ERR_INVALID_STATE, "keyframe not staged");
  StepArgs a;
  memset(&a, 0, sizeof a);
  a.cur = cs;
  a.do_create = 1;
  a.explicit_nbr = 1;
  a.nbr0 = ns;
  a.search_only = 1;
  a.mc = *mc;
  a.n_nbr_req = 1;
  if (unbound_cur) {
    CU(cudaMemcpyAsync(m->d.s.mask_cur, unbound_cur, m->kp_n[cs], cudaMemcpyHostToDevice, ctx->stream));
    a.use_mask_cur = 1;
  }
  if (unbound_nbr) {
    CU(cudaMemcpyAsync(m->d.s.mask_nbr, unbound_nbr, m->kp_n[ns], cudaMemcpyHostToDevice, ctx->stream));
    a.use_mask_nbr = 1;
  }
  rc = launch_steps(ctx, 1, &map, &a);
  if (rc) return rc;
  int cnt = 0;
  CU(cudaMemcpyAsync(&cnt, m->d.s.cand_n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *n_out = cnt;
  if (cnt > cap) return fail(ctx, LM_ERR_CAPACITY, "candidate buffer too small (%d > %d)", cnt, cap);
  std::vector<int> ci(cnt), cj(cnt), cd(cnt);
  if (cnt) {
    CU(cudaMemcpyAsync(ci.data(), m->d.s.cand_i, sizeof(int) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(cj.data(), m->d.s.cand_j, sizeof(int) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(cd.data(), m->d.s.cand_d, sizeof(int) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  for (int k = 0; k < cnt; ++k) {
    out[k].neighbor_kf_id = nbr_kf;
    out[k].kp_index_current = ci[k];
    out[k].kp_index_neighbor = cj[k];
    out[k].distance = cd[k];
    out[k].pad = 0;
  }
  return LM_OK;
}

int lm_fusion_targets(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t n1, int32_t n2, int64_t* out, int32_t cap,
                      int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, true))) return rc;
  if (n1 + n1 * n2 > TMAX) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "n1 + n1*n2 > %d", TMAX);
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_TARGETS;
  a.a = slot;
  a.fc.n1 = n1;
  a.fc.n2 = n2;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  const int T = res[1];
  *n_out = T;
  if (T > cap) return fail(ctx, LM_ERR_CAPACITY, "target buffer too small");
  std::vector<int> t(T);
  if (T) CU(cudaMemcpy(t.data(), m->d.s.targets, sizeof(int) * T, cudaMemcpyDeviceToHost));
  for (int k = 0; k < T; ++k) out[k] = m->ids[t[k]];
  return LM_OK;
}

int lm_fuse_pass(lm_ctx* ctx, int32_t map, const int64_t* point_ids, int32_t n, int64_t target_kf,
                 const lm_fuse_cfg* fc, lm_fuse_action* acts, int32_t act_cap, int32_t* n_act, int64_t* visible,
                 int32_t* n_vis) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, target_kf, &slot, true))) return rc;
  if (n > m->d.s.pts_cap) return fail(ctx, LM_ERR_CAPACITY, "too many points for one pass (%d)", n);
  *n_act = 0;
  *n_vis = 0;
  if (n == 0) return LM_OK;
  std::vector<int> ids(n);
  for (int k = 0; k < n; ++k) ids[k] = (int)point_ids[k];
  CU(cudaMemcpyAsync(m->d.s.pts, ids.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_FUSE_PASS;
  a.a = slot;
  a.n = n;
  a.fc = *fc;
  int res[3];
  if ((rc = run_op(ctx, m, map, a, res, 3))) return rc;
  if (res[0]) return op_status(ctx, res[0], "fuse_pass");
  const int na = res[1];
  if (na > act_cap) return fail(ctx, LM_ERR_CAPACITY, "action buffer too small");
  std::vector<ActRec> ar(na);
  std::vector<int> vf(n);
  if (na) CU(cudaMemcpy(ar.data(), m->d.s.acts, sizeof(ActRec) * na, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(vf.data(), m->d.s.vis_flag, sizeof(int) * n, cudaMemcpyDeviceToHost));
  for (int k = 0; k < na; ++k) {
    acts[k].target_kf_id = m->ids[ar[k].slot];
    acts[k].mp_id_projected = ar[k].pid;
    acts[k].kp_index_hit = ar[k].j;
    acts[k].kind = ar[k].kind;
    acts[k].existing_mp_id = ar[k].other;
  }
  int nv = 0;
  for (int k = 0; k < n; ++k)
    if (vf[k]) visible[nv++] = point_ids[k];
  *n_act = na;
  *n_vis = nv;
  return LM_OK;
}

int lm_apply_fusion(lm_ctx* ctx, int32_t map, const lm_fuse_action* acts, int32_t n, int32_t counts[3]) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  counts[0] = counts[1] = counts[2] = 0;
  if (n == 0) return LM_OK;
  if (n > m->d.s.act_cap) return fail(ctx, LM_ERR_CAPACITY, "too many actions");
  std::vector<ActRec> ar(n);
  for (int k = 0; k < n; ++k) {
    auto it = m->slot_of.find(acts[k].target_kf_id);
    ar[k].slot = it == m->slot_of.end() ? -1 : it->second;
    ar[k].pid = (int)acts[k].mp_id_projected;
    ar[k].j = acts[k].kp_index_hit;
    ar[k].other = (int)acts[k].existing_mp_id;
    ar[k].kind = acts[k].kind;
    if (ar[k].slot < 0 || ar[k].pid < 0) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "action refers to unknown entity");
  }
  CU(cudaMemcpyAsync(m->d.s.acts, ar.data(), sizeof(ActRec) * n, cudaMemcpyHostToDevice, ctx->stream));
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_APPLY;
  a.n = n;
  int res[4];
  if ((rc = run_op(ctx, m, map, a, res, 4))) return rc;
  if (res[0]) return op_status(ctx, res[0], "apply_fusion");
  counts[0] = res[1];
  counts[1] = res[2];
  counts[2] = res[3];
  return LM_OK;
}

int lm_mp_new(lm_ctx* ctx, int32_t map, const double pos[3], const uint8_t desc[32], int64_t first_kf,
              int64_t* id_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_NEW;
  for (int k = 0; k < 3; ++k) a.pos[k] = pos[k];
  memcpy(a.desc, desc, 32);
  a.first_kf = first_kf;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  if (res[0]) return op_status(ctx, res[0], "new_map_point");
  *id_out = res[1];
  return LM_OK;
}

int lm_obs_add(lm_ctx* ctx, int32_t map, int64_t mp, int64_t kf, int32_t kp) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf, &slot, true))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_OBS_ADD;
  a.a = (int)mp;
  a.b = slot;
  a.c = kp;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  return op_status(ctx, res[0], "add_observation");
}

int lm_obs_erase(lm_ctx* ctx, int32_t map, int64_t mp, int64_t kf) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf, &slot, false))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_OBS_ERASE;
  a.a = (int)mp;
  a.b = slot;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  return op_status(ctx, res[0], "erase_observation");
}

int lm_mp_kill(lm_ctx* ctx, int32_t map, int64_t mp) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_KILL;
  a.a = (int)mp;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  return op_status(ctx, res[0], "kill_map_point");
}

int lm_mp_replace(lm_ctx* ctx, int32_t map, int64_t loser, int64_t winner, int32_t* migrated) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_REPLACE;
  a.a = (int)loser;
  a.b = (int)winner;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  if (res[0]) return op_status(ctx, res[0], "replace_map_point");
  if (migrated) *migrated = res[1];
  return LM_OK;
}

int lm_mp_set_counts(lm_ctx* ctx, int32_t map, int64_t mp, int32_t found, int32_t visible) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_SET_COUNTS;
  a.a = (int)mp;
  a.found = found;
  a.visible = visible;
  int res[1];
  return run_op(ctx, m, map, a, res, 1);
}

int lm_cull_keyframes(lm_ctx* ctx, int32_t map, const int64_t* candidates, int32_t n, const lm_kf_cull_cfg* cfg,
                      int64_t* removed, int32_t* n_removed) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (!cfg || n < 0 || (n && !candidates)) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "bad keyframe-cull arguments");
  *n_removed = 0;
  std::vector<long long> ids;
  for (int k = 0; k < n; ++k)
    if (candidates[k] != 0 && m->slot_of.count(candidates[k])) ids.push_back(candidates[k]);  // kf 0: map anchor
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  if (ids.empty()) return LM_OK;
  std::vector<int> slots(ids.size());
  for (size_t k = 0; k < ids.size(); ++k) slots[k] = m->slot_of[ids[k]];
  if ((rc = io_reserve(ctx, m, 2 * sizeof(int) * slots.size()))) return rc;
  CU(cudaMemcpyAsync(m->d_io, slots.data(), sizeof(int) * slots.size(), cudaMemcpyHostToDevice, ctx->stream));
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_KF_CULL;
  a.n = (int)slots.size();
  a.buf = m->d_io;
  a.kc_ratio = cfg->redundancy_ratio;
  a.kc_min_obs = cfg->min_redundant_observers;
  a.kc_tol = cfg->scale_tolerance_levels;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  if (res[0]) return op_status(ctx, res[0], "cull_keyframes");
  const int nr = res[1];
  std::vector<int> rs(nr > 0 ? nr : 1);
  if (nr) CU(cudaMemcpy(rs.data(), (int*)m->d_io + slots.size(), sizeof(int) * nr, cudaMemcpyDeviceToHost));
  for (int k = 0; k < nr; ++k) {
    removed[k] = m->ids[rs[k]];
    m->state[rs[k]] = KF_DEAD;
    if (m->res[rs[k]]) {
      m->res[rs[k]] = 0;
      m->resident--;
    }
  }
  *n_removed = nr;
  return LM_OK;
}

int lm_kf_kill(lm_ctx* ctx, int32_t map, int64_t kf_id) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, true))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_KF_KILL;
  a.a = slot;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  m->state[slot] = KF_DEAD;
  return op_status(ctx, res[0], "kill_keyframe");
}

int lm_covisible_neighbors(lm_ctx* ctx, int32_t map, int64_t kf, int32_t n, int64_t* out, int32_t cap,
                           int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf, &slot, true))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_NEIGHBORS;
  a.a = slot;
  a.n = n < 0 ? 1024 : (n > 1024 ? 1024 : n);
  std::vector<int> res(2 + 1024);
  if ((rc = run_op(ctx, m, map, a, res.data(), 2 + 1024))) return rc;
  const int got = res[1];
  *n_out = got;
  if (got > cap) return fail(ctx, LM_ERR_CAPACITY, "neighbor buffer too small");
  for (int k = 0; k < got; ++k) out[k] = m->ids[res[2 + k]];
  return LM_OK;
}

int lm_ledger_log(lm_ctx* ctx, int32_t map, int64_t first, int64_t* bytes, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  unsigned long long lg[LG_N];
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(lg, m->d.ledger, sizeof lg, cudaMemcpyDeviceToHost));
  long long avail = (long long)lg[LG_SMALL_EVENTS];
  if (avail > LG_LOG_CAP) avail = LG_LOG_CAP;
  long long n = avail - first;
  if (first < 0 || n < 0) n = 0;
  if (n > cap) n = cap;
  if (n_out) *n_out = (int32_t)n;
  if (n) CU(cudaMemcpy(bytes, m->d.lg_log + first, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  return LM_OK;
}

#ifdef LM_DIAG
// diagnostics build only: read (and clear) the device diagnostic words
int lm_debug_diag(uint64_t* out, int n) {
  if (n > 64) n = 64;
  if (cudaDeviceSynchronize() != cudaSuccess) return LM_ERR_CUDA;
  if (cudaMemcpyFromSymbol(out, lm::g_diag, n * sizeof(uint64_t)) != cudaSuccess) return LM_ERR_CUDA;
  static const unsigned long long zero[64] = {0};
  cudaMemcpyToSymbol(lm::g_diag, zero, sizeof(zero));
  return LM_OK;
}
#endif

int lm_debug_corrupt(lm_ctx* ctx, int32_t map, int32_t what, int64_t a, int64_t b, int32_t delta) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  OpArgs o;
  memset(&o, 0, sizeof o);
  o.op = OP_CORRUPT;
  o.n = what;
  o.c = delta;
  if (what == 0) {
    int next = 0;
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
    if (a < 0 || a >= next || b < 0 || b >= m->d.L) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "bad counter cell");
    o.a = (int)a;
    o.b = (int)b;
  } else {
    int sa, sb;
    if ((rc = slot_of(ctx, m, a, &sa, false)) || (rc = slot_of(ctx, m, b, &sb, false))) return rc;
    o.a = sa;
    o.b = sb;
  }
  int res[1];
  if ((rc = run_op(ctx, m, map, o, res, 1))) return rc;
  return op_status(ctx, res[0], "corrupt");
}

int lm_ledger_add(lm_ctx* ctx, int32_t map, int64_t naive_bytes, int32_t small_stage_triangulation,
                  int64_t small_bytes, int32_t small_events) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (naive_bytes < 0 || small_bytes < 0 || small_events < 0 || small_events > 1)
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "transfer size must be non-negative");
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_LEDGER_ADD;
  a.v0 = naive_bytes;
  a.v1 = small_bytes;
  a.n = small_events;
  a.b = small_stage_triangulation ? 1 : 0;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  return op_status(ctx, res[0], "ledger");
}

int lm_audit(lm_ctx* ctx, int32_t map, lm_audit_record* out, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if ((rc = refresh(ctx, m, map))) return rc;  // clean lists are sorted (not required, but cheap)
  int next = 0;
  CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
  const size_t K = m->d.kf_cap;
  const int rcap = 1 << 16;
  void* scratch = nullptr;
  CU(cudaMalloc(&scratch, sizeof(int) * (K * K + 4) + sizeof(int4) * rcap));
  AuditOut O;
  O.count = (int*)scratch;
  O.expect = O.count + 4;
  O.rec = (int4*)(O.expect + K * K);
  O.cap = rcap;
  cudaStream_t st = ctx->stream;
  int rc2 = LM_OK;
  do {
    if (cudaMemsetAsync(scratch, 0, sizeof(int) * (K * K + 4), st) != cudaSuccess) { rc2 = LM_ERR_CUDA; break; }
    if (next) k_audit_points<<<(next + 255) / 256, 256, 0, st>>>(m->d, O, next);
    if (m->n_slots) {
      k_audit_slots<<<dim3((m->d.kpkf_max + 255) / 256, m->n_slots < 1024 ? m->n_slots : 1024), 256, 0, st>>>(
          m->d, O, m->n_slots, next);
      const long long np = (long long)m->n_slots * m->n_slots;
      const int blocks = (int)((np + 255) / 256 < 4096 ? (np + 255) / 256 : 4096);
      k_audit_covis<<<blocks, 256, 0, st>>>(m->d, O, m->n_slots);
    }
    ctx->launches += 3;
  } while (0);
  int total = 0;
  std::vector<int4> rec;
  if (rc2 == LM_OK && cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess &&
      cudaMemcpy(&total, O.count, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess) {
    const int got = total < rcap ? total : rcap;
    rec.resize(got > 0 ? got : 1);
    if (got) cudaMemcpy(rec.data(), O.rec, sizeof(int4) * got, cudaMemcpyDeviceToHost);
    rec.resize(got);
  } else {
    rc2 = LM_ERR_CUDA;
  }
  cudaFree(scratch);
  if (rc2) return fail(ctx, rc2, "audit kernels failed");
  if (n_out) *n_out = total;
  const int w = (int)rec.size() < cap ? (int)rec.size() : cap;
  for (int k = 0; k < w; ++k) {  // slots -> keyframe ids
    const int4 r = rec[k];
    lm_audit_record& o = out[k];
    o.code = r.x;
    switch (r.x) {
      case AV_OBS_DEAD_KF: o.mp = r.y; o.kf_a = m->ids[r.z]; o.kf_b = -1; o.kp = -1; break;
      case AV_BIND_MISMATCH: o.mp = r.y; o.kf_a = m->ids[r.z]; o.kf_b = -1; o.kp = r.w; break;
      case AV_SLOT_DEAD:
      case AV_SLOT_NOT_OBS: o.mp = r.w; o.kf_a = m->ids[r.y]; o.kf_b = -1; o.kp = r.z; break;
      case AV_COVIS: o.mp = -1; o.kf_a = m->ids[r.y]; o.kf_b = m->ids[r.z]; o.kp = -1; break;
      default: o.mp = r.y; o.kf_a = -1; o.kf_b = -1; o.kp = -1;
    }
  }
  return LM_OK;
}

int lm_ledger(lm_ctx* ctx, int32_t map, lm_ledger_t* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  unsigned long long lg[LG_N];
  CU(cudaMemcpyAsync(lg, m->d.ledger, sizeof lg, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  out->persistent_bytes_up = (int64_t)lg[LG_PERSIST];
  out->naive_bytes_up = (int64_t)lg[LG_NAIVE];
  out->small_bytes_triangulation = (int64_t)lg[LG_SMALL_TRI];
  out->small_bytes_fusion = (int64_t)lg[LG_SMALL_FUSE];
  out->small_transfer_events = (int64_t)lg[LG_SMALL_EVENTS];
  out->evictions = (int64_t)lg[LG_EVICT];
  return LM_OK;
}

static int refresh(lm_ctx* ctx, HostMap* m, int map) {
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_REFRESH;
  int res[1];
  int rc = run_op(ctx, m, map, a, res, 1);
  if (rc) return rc;
  return res[0] ? op_status(ctx, res[0], "refresh") : LM_OK;
}

int lm_export_keyframes(lm_ctx* ctx, int32_t map, int64_t* kf_id, int32_t* state, int32_t* kp_off, int32_t* kp_n,
                        int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  const int n = m->n_slots;
  *n_out = n;
  if (n > cap) return fail(ctx, LM_ERR_CAPACITY, "keyframe buffer too small");
  for (int s = 0; s < n; ++s) {
    kf_id[s] = m->ids[s];
    state[s] = m->state[s];
    kp_off[s] = m->kp_off[s];
    kp_n[s] = m->kp_n[s];
  }
  return LM_OK;
}

int lm_export_bindings(lm_ctx* ctx, int32_t map, int32_t* bind, int32_t cap) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (cap < m->kp_head) return fail(ctx, LM_ERR_CAPACITY, "binding buffer too small");
  CU(cudaStreamSynchronize(ctx->stream));
  if (m->kp_head) CU(cudaMemcpy(bind, m->d.kbind, sizeof(int) * m->kp_head, cudaMemcpyDeviceToHost));
  return LM_OK;
}

int lm_export_points(lm_ctx* ctx, int32_t map, int32_t n, double* pos, uint8_t* rep, uint8_t* alive, int32_t* found,
                     int32_t* visible, int32_t* nobs, int32_t* counts, int64_t* obs_kf, int32_t* obs_kp,
                     int32_t obs_cap) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if ((rc = refresh(ctx, m, map))) return rc;
  if (n <= 0) return LM_OK;
  const DevMap& d = m->d;
  CU(cudaMemcpy(pos, d.pos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(rep, d.rep, 32 * (size_t)n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(alive, d.alive, n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(found, d.found, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(visible, d.visible, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(nobs, d.nobs, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(counts, d.counts, sizeof(int) * n * d.L, cudaMemcpyDeviceToHost));
  std::vector<int> off(n);
  CU(cudaMemcpy(off.data(), d.ooff, sizeof(int) * n, cudaMemcpyDeviceToHost));
  int used = 0;
  CU(cudaMemcpy(&used, d.scal + SC_OBS_HEAD, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int2> pool(used > 0 ? used : 1);
  if (used) CU(cudaMemcpy(pool.data(), d.obs, sizeof(int2) * used, cudaMemcpyDeviceToHost));
  long long tot = 0;
  for (int i = 0; i < n; ++i) tot += nobs[i];
  if (tot > obs_cap) return fail(ctx, LM_ERR_CAPACITY, "observation buffer too small (%lld)", tot);
  int w = 0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < nobs[i]; ++k) {
      const int2 e = pool[off[i] + k];
      obs_kf[w] = m->ids[e.x];
      obs_kp[w] = e.y;
      ++w;
    }
  return LM_OK;
}

int lm_export_covis(lm_ctx* ctx, int32_t map, int32_t* w, int32_t cap) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  const size_t K = m->d.kf_cap;
  if ((size_t)cap < K * K) return fail(ctx, LM_ERR_CAPACITY, "covis buffer too small");
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(w, m->d.covis, sizeof(int) * K * K, cudaMemcpyDeviceToHost));
  return LM_OK;
}

int lm_recent_export(lm_ctx* ctx, int32_t map, int64_t* ids, int32_t* born, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int n = 0;
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(&n, m->d.scal + SC_RECENT_N, sizeof(int), cudaMemcpyDeviceToHost));
  *n_out = n;
  if (n > cap) return fail(ctx, LM_ERR_CAPACITY, "recent buffer too small");
  std::vector<int> id(n);
  if (n) {
    CU(cudaMemcpy(id.data(), m->d.recent_id, sizeof(int) * n, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(born, m->d.recent_born, sizeof(int) * n, cudaMemcpyDeviceToHost));
  }
  for (int k = 0; k < n; ++k) ids[k] = id[k];
  return LM_OK;
}

int lm_recent_import(lm_ctx* ctx, int32_t map, const int64_t* ids, const int32_t* born, int32_t n) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (n > m->d.recent_cap) return fail(ctx, LM_ERR_CAPACITY, "recent list too long");
  std::vector<int> id(n);
  for (int k = 0; k < n; ++k) id[k] = (int)ids[k];
  CU(cudaStreamSynchronize(ctx->stream));
  if (n) {
    CU(cudaMemcpy(m->d.recent_id, id.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(m->d.recent_born, born, sizeof(int) * n, cudaMemcpyHostToDevice));
  }
  CU(cudaMemcpy(m->d.scal + SC_RECENT_N, &n, sizeof(int), cudaMemcpyHostToDevice));
  return LM_OK;
}

// ------------------------------------------------------------------- store / LBA write-back / import


int lm_kf_upload(lm_ctx* ctx, int32_t map, int64_t kf_id) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, false))) return rc;
  if (m->state[slot] == KF_STAGED)
    return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld is staged, not inserted", (long long)kf_id);
  if (m->res[slot]) return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld already resident", (long long)kf_id);
  if (m->caps.store_capacity > 0 && m->resident >= m->caps.store_capacity)
    return fail(ctx, LM_ERR_CAPACITY, "store capacity %d exceeded; size the pre-allocation", m->caps.store_capacity);
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_UPLOAD;
  a.a = slot;
  if ((rc = run_op_async(ctx, m, map, a))) return rc;  // validated above; cannot fail on the device
  m->res[slot] = 1;
  m->resident++;
  return LM_OK;
}

int lm_kf_evict(lm_ctx* ctx, int32_t map, int64_t kf_id) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  auto it = m->slot_of.find(kf_id);
  if (it == m->slot_of.end() || !m->res[it->second])
    return fail(ctx, LM_ERR_INVALID_ARGUMENT, "keyframe %lld is not resident", (long long)kf_id);
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_EVICT;
  a.a = it->second;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  m->res[it->second] = 0;
  m->resident--;
  return op_status(ctx, res[0], "evict_keyframe");
}

int lm_map_enforce_residency(lm_ctx* ctx, int32_t map, int32_t enforce) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  const int v = enforce ? 0 : 1;
  CU(cudaMemcpyAsync(m->d.scal + SC_NORES, &v, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return LM_OK;
}

int lm_kf_resident(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t* resident, int32_t* count) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  auto it = m->slot_of.find(kf_id);
  if (resident) *resident = it != m->slot_of.end() && m->res[it->second];
  if (count) *count = m->resident;
  return LM_OK;
}

int lm_kf_set_pose(lm_ctx* ctx, int32_t map, int64_t kf_id, const double quat[4], const double trans[3]) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (!quat || !trans) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "pose arrays required");
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, false))) return rc;
  if (m->state[slot] == KF_DEAD) return fail(ctx, LM_ERR_INVALID_STATE, "keyframe %lld is dead", (long long)kf_id);
  for (int k = 0; k < 4; ++k)
    if (!std::isfinite(quat[k])) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "non-finite quaternion");
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_SET_POSE;
  a.a = slot;
  double* q = a.pose;
  double *R = q + 4, *t = q + 13, *Cc = q + 16, *P = q + 19;
  for (int k = 0; k < 4; ++k) q[k] = quat[k];
  for (int k = 0; k < 3; ++k) t[k] = trans[k];
  // the same host code as staging (tables bit-identical to a fresh stage of the new pose);
  // the camera is the slot's (read back from the host mirror of the staged record)
  double cam[6];
  CU(cudaMemcpy(cam, m->d.cam + 6 * slot, sizeof cam, cudaMemcpyDeviceToHost));
  quat_to_rot(q, R);
  camera_center(R, t, Cc);
  proj_matrix(cam[0], cam[1], cam[2], cam[3], R, t, P);
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  return op_status(ctx, res[0], "set_pose");
}

int lm_mp_patch_positions(lm_ctx* ctx, int32_t map, int32_t n, const int64_t* ids, const double* pos) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (n < 0 || (n && (!ids || !pos))) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "ids/pos required");
  if (n == 0) return LM_OK;
  int next = 0;
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<unsigned char> alive(next > 0 ? next : 1);
  if (next) CU(cudaMemcpy(alive.data(), m->d.alive, next, cudaMemcpyDeviceToHost));
  std::vector<char> buf(32 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    if (ids[k] < 0 || ids[k] >= next) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown map point %lld", (long long)ids[k]);
    if (!alive[ids[k]]) return fail(ctx, LM_ERR_INVALID_STATE, "map point %lld is dead", (long long)ids[k]);
    const int id = (int)ids[k];
    memcpy(&buf[32 * (size_t)k], &id, 4);
    memcpy(&buf[32 * (size_t)k + 8], pos + 3 * (size_t)k, 24);
  }
  if ((rc = io_reserve(ctx, m, buf.size()))) return rc;
  CU(cudaMemcpyAsync(m->d_io, buf.data(), buf.size(), cudaMemcpyHostToDevice, ctx->stream));
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_PATCH_POS;
  a.n = n;
  a.buf = m->d_io;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  return op_status(ctx, res[0], "patch_positions");
}

int lm_mp_get(lm_ctx* ctx, int32_t map, int64_t mp, lm_point_record* out, int64_t* obs_kf, int32_t* obs_kp,
              int32_t obs_cap) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (!out) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "output record required");
  int next = 0;
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
  if (mp < 0 || mp >= next) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown map point %lld", (long long)mp);
  const size_t bytes = sizeof(PointRec) + sizeof(int2) * (size_t)m->d.kf_cap;
  if ((rc = io_reserve(ctx, m, bytes))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_MP_GET;
  a.a = (int)mp;
  a.buf = m->d_io;
  int res[1];
  if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  std::vector<char> h(sizeof(PointRec));
  CU(cudaMemcpy(h.data(), m->d_io, sizeof(PointRec), cudaMemcpyDeviceToHost));
  const PointRec* r = (const PointRec*)h.data();
  std::vector<int2> o(r->nobs > 0 ? r->nobs : 1);
  if (r->nobs) CU(cudaMemcpy(o.data(), (char*)m->d_io + sizeof(PointRec), sizeof(int2) * r->nobs, cudaMemcpyDeviceToHost));
  memcpy(out->pos, r->pos, 24);
  memcpy(out->rep, r->rep, 32);
  out->first_kf_id = r->first_kf;
  out->alive = r->alive;
  out->found = r->found;
  out->visible = r->visible;
  out->nobs = r->nobs;
  for (int l = 0; l < 16; ++l) out->counts[l] = r->counts[l];
  if (r->nobs > obs_cap) return fail(ctx, LM_ERR_CAPACITY, "observation buffer too small (%d)", r->nobs);
  for (int k = 0; k < r->nobs; ++k) {
    if (obs_kf) obs_kf[k] = m->ids[o[k].x];
    if (obs_kp) obs_kp[k] = o[k].y;
  }
  return op_status(ctx, res[0], "mp_get");
}

int lm_mp_alive(lm_ctx* ctx, int32_t map, int32_t n, const int64_t* ids, uint8_t* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (n <= 0) return LM_OK;
  int next = 0;
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
  // ids are probation entries: a contiguous window of recent ids, so one range copy
  long long lo = next, hi = -1;
  for (int k = 0; k < n; ++k) {
    if (ids[k] < 0 || ids[k] >= next) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "unknown map point %lld", (long long)ids[k]);
    lo = ids[k] < lo ? ids[k] : lo;
    hi = ids[k] > hi ? ids[k] : hi;
  }
  std::vector<unsigned char> a(hi - lo + 1);
  CU(cudaMemcpy(a.data(), m->d.alive + lo, a.size(), cudaMemcpyDeviceToHost));
  for (int k = 0; k < n; ++k) out[k] = a[ids[k] - lo];
  return LM_OK;
}

int lm_kf_bindings(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* out, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, false))) return rc;
  const int n = m->kp_n[slot];
  if (n_out) *n_out = n;
  if (n > cap) return fail(ctx, LM_ERR_CAPACITY, "binding buffer too small");
  std::vector<int> b(n > 0 ? n : 1);
  CU(cudaStreamSynchronize(ctx->stream));
  if (n) CU(cudaMemcpy(b.data(), m->d.kbind + m->kp_off[slot], sizeof(int) * n, cudaMemcpyDeviceToHost));
  for (int k = 0; k < n; ++k) out[k] = b[k];
  return LM_OK;
}

int lm_bound_points(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* out, int32_t cap, int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, false))) return rc;
  if ((rc = io_reserve(ctx, m, sizeof(int) * (size_t)(m->kp_n[slot] + 1)))) return rc;
  OpArgs a;
  memset(&a, 0, sizeof a);
  a.op = OP_BOUND;
  a.a = slot;
  a.buf = m->d_io;
  int res[2];
  if ((rc = run_op(ctx, m, map, a, res, 2))) return rc;
  const int P = res[1];
  if (n_out) *n_out = P;
  if (P > cap) return fail(ctx, LM_ERR_CAPACITY, "point buffer too small");
  std::vector<int> b(P > 0 ? P : 1);
  if (P) CU(cudaMemcpy(b.data(), m->d_io, sizeof(int) * P, cudaMemcpyDeviceToHost));
  for (int k = 0; k < P; ++k) out[k] = b[k];
  return LM_OK;
}

int lm_covis_row(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* kf_ids, int32_t* weights, int32_t cap,
                 int32_t* n_out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  int slot;
  if ((rc = slot_of(ctx, m, kf_id, &slot, false))) return rc;
  const int K = m->d.kf_cap;
  std::vector<int> row(K);
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(row.data(), m->d.covis + (size_t)slot * K, sizeof(int) * K, cudaMemcpyDeviceToHost));
  int n = 0;
  for (int s = 0; s < m->n_slots; ++s)
    if (row[s] != 0 && s != slot) {
      if (n < cap) {
        kf_ids[n] = m->ids[s];
        weights[n] = row[s];
      }
      ++n;
    }
  if (n_out) *n_out = n;
  if (n > cap) return fail(ctx, LM_ERR_CAPACITY, "covisibility buffer too small");
  return LM_OK;
}

// Import a whole reference map state (MapModel + DeviceStore ledger + probation list) into an
// empty map: points first (ids 0..n-1, no observations), then every keyframe staged with its
// bindings and inserted in the given order, which registers the observations exactly as
// insert_keyframe does (mapmodel.py:185-199: sorted lists, per-level counters, covisibility
// as the shared-point counts), then dead keyframes tombstoned, residency, ledger and the
// probation list set. Representative descriptors are recomputed (a pure function of the
// observation list, equal to the reference's stored one).
int lm_import_snapshot(lm_ctx* ctx, int32_t map, const lm_snapshot* S) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  if (!S || S->n_kf < 0 || S->n_points < 0) return fail(ctx, LM_ERR_INVALID_ARGUMENT, "bad snapshot");
  {
    int next = 0;
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(&next, m->d.scal + SC_NEXT_ID, sizeof(int), cudaMemcpyDeviceToHost));
    if (m->n_slots || next) return fail(ctx, LM_ERR_INVALID_STATE, "import needs an empty map (lm_map_reset)");
  }
  if (S->n_points > m->d.mp_cap) return fail(ctx, LM_ERR_CAPACITY, "snapshot has %d points, map capacity %d",
                                              S->n_points, m->d.mp_cap);
  if (S->n_points) {
    std::vector<char> buf(96 * (size_t)S->n_points, 0);
    for (int i = 0; i < S->n_points; ++i) {
      char* e = &buf[96 * (size_t)i];
      memcpy(e, S->pos + 3 * (size_t)i, 24);
      memcpy(e + 32, S->rep + 32 * (size_t)i, 32);
      const long long fk = S->first_kf ? (long long)S->first_kf[i] : -1;
      memcpy(e + 64, &fk, 8);
      memcpy(e + 72, S->found + i, 4);
      memcpy(e + 76, S->visible + i, 4);
      e[80] = S->alive[i] ? 1 : 0;
    }
    if ((rc = io_reserve(ctx, m, buf.size()))) return rc;
    CU(cudaMemcpyAsync(m->d_io, buf.data(), buf.size(), cudaMemcpyHostToDevice, ctx->stream));
    OpArgs a;
    memset(&a, 0, sizeof a);
    a.op = OP_IMPORT_POINTS;
    a.n = S->n_points;
    a.buf = m->d_io;
    int res[1];
    if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
    if (res[0]) return op_status(ctx, res[0], "import points");
  }
  size_t off = 0;
  for (int k = 0; k < S->n_kf; ++k) {
    const int n = S->kp_n[k];
    const bool live = S->kf_alive[k] != 0;
    if ((rc = lm_kf_stage(ctx, map, S->kf_id[k], S->quat + 4 * (size_t)k, S->trans + 3 * (size_t)k,
                          S->cam + 6 * (size_t)k, n, S->u + off, S->v + off, S->level + off, S->desc + 32 * off,
                          live ? S->bindings + off : nullptr)))
      return rc;
    if ((rc = lm_kf_insert(ctx, map, S->kf_id[k]))) return rc;
    if (!live && (rc = lm_kf_kill(ctx, map, S->kf_id[k]))) return rc;
    if (S->kf_resident && S->kf_resident[k] && (rc = lm_kf_upload(ctx, map, S->kf_id[k]))) return rc;
    off += n;
  }
  // representative descriptors and sorted lists: refresh every dirty point now; then every
  // point's view-geometry cache (the stages expect clean points to carry valid caches)
  if ((rc = refresh(ctx, m, map))) return rc;
  {
    OpArgs a;
    memset(&a, 0, sizeof a);
    a.op = OP_GEO_ALL;
    int res[1];
    if ((rc = run_op(ctx, m, map, a, res, 1))) return rc;
  }
  unsigned long long lg[LG_N] = {0};
  lg[LG_PERSIST] = S->ledger.persistent_bytes_up;
  lg[LG_NAIVE] = S->ledger.naive_bytes_up;
  lg[LG_SMALL_TRI] = S->ledger.small_bytes_triangulation;
  lg[LG_SMALL_FUSE] = S->ledger.small_bytes_fusion;
  lg[LG_SMALL_EVENTS] = S->ledger.small_transfer_events;
  lg[LG_EVICT] = S->ledger.evictions;
  CU(cudaMemcpy(m->d.ledger, lg, sizeof lg, cudaMemcpyHostToDevice));
  if (S->n_recent && (rc = lm_recent_import(ctx, map, S->recent_id, S->recent_born, S->n_recent))) return rc;
  return LM_OK;
}

// ------------------------------------------------------------------- measurement
__global__ void k_rewind_state(DevMap M, int n_slots) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += gridDim.x * blockDim.x)
    if (M.kf_state[s] != KF_FREE) M.kf_state[s] = KF_STAGED;
}

int lm_map_rewind(lm_ctx* ctx, int32_t map) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  DevMap& d = m->d;
  const size_t K = d.kf_cap, MP = d.mp_cap;
  cudaStream_t st = ctx->stream;
  CU(cudaMemsetAsync(d.covis, 0, sizeof(int) * K * K, st));
  CU(cudaMemsetAsync(d.kf_res, 0, K, st));
  CU(cudaMemsetAsync(d.alive, 0, MP, st));
  CU(cudaMemsetAsync(d.nobs, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.ocap, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.counts, 0, sizeof(int) * MP * d.L, st));
  CU(cudaMemsetAsync(d.dirty, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.gval, 0, MP, st));
  CU(cudaMemsetAsync(d.hit, 0xff, sizeof(int2) * MP, st));
  CU(cudaMemsetAsync(d.ver, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.scal, 0, sizeof(int) * SC_N, st));
  CU(cudaMemsetAsync(d.ledger, 0, sizeof(unsigned long long) * LG_N, st));
  CU(cudaMemsetAsync(m->d_totals, 0, sizeof(lm_step_stats), st));
  CU(cudaMemsetAsync(d.res_pt, 0xff, sizeof(unsigned long long) * MP, st));
  CU(cudaMemsetAsync(d.res_slot, 0xff, sizeof(unsigned long long) * d.kp_cap, st));
  CU(cudaMemsetAsync(d.res_ex, 0xff, sizeof(unsigned long long) * MP, st));
  CU(cudaMemsetAsync(d.res_pair, 0xff, sizeof(unsigned long long) * RES_PAIR, st));
  CU(cudaMemsetAsync(d.grp_head, 0, sizeof(unsigned long long) * MP, st));
  CU(cudaMemsetAsync(d.s.rmark, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.s.die, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.s.itag, 0, sizeof(int) * d.s.act_cap, st));
  CU(cudaMemsetAsync(d.mrg, 0, sizeof(int2) * MP, st));
  CU(cudaMemsetAsync(d.s.hreg, 0, sizeof(int) * MP, st));
  CU(cudaMemsetAsync(d.sp_tag, 0, sizeof(int) * MP, st));
  if (m->kp_head) CU(cudaMemsetAsync(d.kbind, 0xff, sizeof(int) * m->kp_head, st));
  if (m->n_slots) {
    k_rewind_state<<<(m->n_slots + 255) / 256, 256, 0, st>>>(d, m->n_slots);
    CHECK_LAUNCH();
  }
  CU(cudaStreamSynchronize(st));
  for (int s = 0; s < m->n_slots; ++s)
    if (m->state[s] != KF_FREE) m->state[s] = KF_STAGED;
  std::fill(m->res.begin(), m->res.end(), 0);
  m->resident = 0;
  return LM_OK;
}

int lm_timer_start(lm_ctx* ctx) {
  if (!ctx->t0) {
    CU(cudaEventCreate(&ctx->t0));
    CU(cudaEventCreate(&ctx->t1));
  }
  CU(cudaEventRecord(ctx->t0, ctx->stream));
  return LM_OK;
}

int lm_timer_stop(lm_ctx* ctx, float* ms) {
  CU(cudaEventRecord(ctx->t1, ctx->stream));
  CU(cudaEventSynchronize(ctx->t1));
  CU(cudaEventElapsedTime(ms, ctx->t0, ctx->t1));
  return LM_OK;
}

int lm_timer_start_joint(lm_ctx* ctx, lm_ctx* other) {
  // start on ctx's stream; other's stream waits for it, so other's later work is inside
  int rc = lm_timer_start(ctx);
  if (rc) return rc;
  if (other && other != ctx) CU(cudaStreamWaitEvent(other->stream, ctx->t0, 0));
  return LM_OK;
}

int lm_timer_stop_joint(lm_ctx* ctx, lm_ctx* other, float* ms) {
  // elapsed from ctx's start event to the later of the two streams' stop events
  if (!other || other == ctx) return lm_timer_stop(ctx, ms);
  if (!other->t0) {
    CU(cudaEventCreate(&other->t0));
    CU(cudaEventCreate(&other->t1));
  }
  CU(cudaEventRecord(ctx->t1, ctx->stream));
  CU(cudaEventRecord(other->t1, other->stream));
  CU(cudaEventSynchronize(ctx->t1));
  CU(cudaEventSynchronize(other->t1));
  float a = 0, b = 0;
  CU(cudaEventElapsedTime(&a, ctx->t0, ctx->t1));
  CU(cudaEventElapsedTime(&b, ctx->t0, other->t1));
  *ms = a > b ? a : b;
  return LM_OK;
}

int lm_timer_start_multi(lm_ctx* const* ctxs, int32_t n) {
  if (!ctxs || n < 1 || !ctxs[0]) return LM_ERR_INVALID_ARGUMENT;
  lm_ctx* ctx = ctxs[0];
  int rc = lm_timer_start(ctx);
  if (rc) return rc;
  for (int i = 1; i < n; ++i) CU(cudaStreamWaitEvent(ctxs[i]->stream, ctxs[0]->t0, 0));
  return LM_OK;
}

int lm_timer_stop_multi(lm_ctx* const* ctxs, int32_t n, float* ms) {
  if (!ctxs || n < 1 || !ctxs[0] || !ms) return LM_ERR_INVALID_ARGUMENT;
  lm_ctx* ctx = ctxs[0];
  float best = 0;
  for (int i = 0; i < n; ++i) {
    lm_ctx* c = ctxs[i];
    if (!c->t0) {
      CU(cudaEventCreate(&c->t0));
      CU(cudaEventCreate(&c->t1));
    }
    CU(cudaEventRecord(c->t1, c->stream));
  }
  for (int i = 0; i < n; ++i) {
    CU(cudaEventSynchronize(ctxs[i]->t1));
    float t = 0;
    CU(cudaEventElapsedTime(&t, ctxs[0]->t0, ctxs[i]->t1));
    best = t > best ? t : best;
  }
  *ms = best;
  return LM_OK;
}

int lm_flush_l2(lm_ctx* ctx, int64_t bytes) {
  if (bytes <= 0) return LM_OK;
  if ((size_t)bytes > ctx->flush_bytes) {
    if (ctx->flush_buf) CU(cudaFree(ctx->flush_buf));
    CU(cudaMalloc(&ctx->flush_buf, (size_t)bytes));
    ctx->flush_bytes = (size_t)bytes;
  }
  CU(cudaMemsetAsync(ctx->flush_buf, (int)(ctx->launches & 0xff), (size_t)bytes, ctx->stream));
  return LM_OK;
}

int lm_totals_fetch(lm_ctx* ctx, int32_t map, lm_step_stats* out) {
  HostMap* m;
  int rc = check_map(ctx, map, &m);
  if (rc) return rc;
  CU(cudaMemcpyAsync(out, m->d_totals, sizeof(lm_step_stats), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return LM_OK;
}

int64_t lm_launch_count(lm_ctx* ctx) { return ctx ? ctx->launches : -1; }

int lm_profile_enable(lm_ctx* ctx, int32_t on) {
  ctx->prof = on != 0;
  return LM_OK;
}

int lm_profile_read(lm_ctx* ctx, double ms[16], int64_t launches[16]) {
  CU(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < 16; ++k) {
    ms[k] = 0;
    launches[k] = 0;
  }
  for (auto& evs : ctx->prof_steps) {
    for (size_t k = 0; k + 1 < evs.size() && k < 16; ++k) {
      float t = 0;
      CU(cudaEventElapsedTime(&t, evs[k], evs[k + 1]));
      ms[k] += t;
      launches[k] += 1;
    }
    for (cudaEvent_t ev : evs) ctx->prof_pool.push_back(ev);
  }
  ctx->prof_steps.clear();
  return LM_OK;
}

__global__ void k_popc_bench(unsigned* out, int iters, unsigned key) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3 + 1, a2 = a0 * 5 + 2, a3 = a0 * 7 + 3;
  unsigned a4 = a0 * 11 + 4, a5 = a0 * 13 + 5, a6 = a0 * 17 + 6, a7 = a0 * 19 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 += __popc(a0 ^ key); a1 += __popc(a1 ^ key); a2 += __popc(a2 ^ key); a3 += __popc(a3 ^ key);
    a4 += __popc(a4 ^ key); a5 += __popc(a5 ^ key); a6 += __popc(a6 ^ key); a7 += __popc(a7 ^ key);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

int lm_bench_popc(lm_ctx* ctx, double* popc_per_s) {
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  unsigned* out;
  CU(cudaMalloc(&out, sizeof(unsigned) * blocks * threads));
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  k_popc_bench<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0x9e3779b9u);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CU(cudaEventRecord(a, ctx->stream));
    k_popc_bench<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0x9e3779b9u + rep);
    CU(cudaEventRecord(b, ctx->stream));
    CU(cudaEventSynchronize(b));
    float t;
    CU(cudaEventElapsedTime(&t, a, b));
    best = t < best ? t : best;
  }
  CU(cudaFree(out));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *popc_per_s = (double)blocks * threads * iters * 8 / (best * 1e-3);
  return LM_OK;
}

// ------------------------------------------------------------------- host math (CPU tests)
int lm_host_fundamental(const double qa[4], const double ta[3], const double qb[4], const double tb[3],
                        const double cam_a[4], const double cam_b[4], double F[9]) {
  return fundamental(qa, ta, qb, tb, cam_a, cam_b, F) ? LM_OK : LM_ERR_DEGENERATE;
}

int lm_host_projection(const double quat[4], const double trans[3], const double cam[4], double R[9], double C[3],
                       double P[12]) {
  quat_to_rot(quat, R);
  camera_center(R, trans, C);
  proj_matrix(cam[0], cam[1], cam[2], cam[3], R, trans, P);
  return LM_OK;
}

int lm_host_triangulate(const double Pa[12], const double Pb[12], const double Ca[3], const double Cb[3],
                        const double pix[4], double X[3]) {
  return triangulate(Pa, Pb, Ca, Cb, pix[0], pix[1], pix[2], pix[3], X) ? LM_OK : LM_ERR_DEGENERATE;
}

}  // extern "C"
