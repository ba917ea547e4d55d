// lm_kernels.cuh -- the per-keyframe kernels of the hot path (sm_100a).
//
// One step for a batch of maps (blockIdx.{y,z} or blockIdx.x selects the map):
//   k_insert   insert a staged keyframe (state, ledger, pre-bound slots)
//   k_cull     recent map-point culling (culling.py:28-59), one CTA per map
//   k_select   covisible neighbours + recency padding + F per pair (triangulation.py:219-232)
//   k_prep     level-bucketed unbound keypoint lists per (current | neighbour)
//   k_match    popcount Hamming x epipolar search, tile of current keypoints x one neighbour
//              (triangulation.py:117-136), then one-to-one via 64-bit atomicMin (63-77)
//   k_tri      candidate compaction in current-index order + fused DLT + creation gates
//   k_commit   winner = lowest neighbour rank whose candidate passes; ids by block scan in
//              (rank, i) order; point / binding / counter / covisibility writes (257-299)
//   k_fuse_*   SearchAndFuse (fusion.py:307-347):
//              targets    collect_fusion_targets + forward point list (1 CTA / map)
//              geo        stale descriptors + geometry rows of the forward points (warp / point)
//              gather     forward gather-all, thread per (target, point)
//              apply      forward apply-all, reservation rounds on a CTA cluster per map
//              refresh    every point the forward apply touched (warp / point)
//              spec*      every reverse pass's items, speculatively (thread per item)
//              post       post-ADD states of the speculative reverse ADDs (warp / point)
//              rev        the ordered reverse passes (1 CTA / map), re-evaluating only what an
//                         acting pass touched
//              visible    the reverse passes' visible counters (thread per item)
#pragma once
#include <cooperative_groups.h>

#include "lm_map.cuh"
#include "lm_math.cuh"

namespace lm {

namespace cg = cooperative_groups;

struct StepArgs {
  int map;            // index into the context's map table
  int cur;            // current keyframe slot
  int n_nbr_req;      // neighbor_count
  int do_insert, do_cull, do_create, do_fuse;
  int do_upload;      // with do_insert: also DeviceStore.upload_keyframe (residency + ledger)
  int select_early;   // k_select may run concurrently with k_cull (see k_select)
  int prebound;       // the inserted keyframe was staged with pre-bound slots
  int processed;      // pipeline._processed
  int explicit_nbr;   // lm_search: neighbour list given (nbr0), masks optional
  int nbr0;
  int use_mask_cur, use_mask_nbr;
  int search_only;    // lm_search: stop after candidate compaction
  lm_match_cfg mc;
  lm_gate_cfg gc;
  lm_fuse_cfg fc;
  lm_cull_cfg cc;
};

// ---------------------------------------------------------------------------------- helpers

// programmatic dependent launch: a step kernel first waits for its predecessor's completion
// (and memory), then lets its own successor be scheduled, so each launch's dispatch overlaps
// the previous kernel instead of following it (no-ops when launched without the attribute)
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

__device__ __forceinline__ long long gtime() {  // ns, device-wide clock
#ifdef LM_NO_PHASE_TIMERS
  return 0;
#else
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
#endif
}

// phase-timer reads of the kernels instantiated twice: with timers (P, the library's profile
// pass: lm_profile_enable) and without (every other launch). The timer-free instantiation
// measured 0.9% faster on C2 than one that reads the timer in every launch.
template <bool P>
__device__ __forceinline__ long long gtime_p() {
  return P ? gtime() : 0;
}

template <int BLOCK>
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < BLOCK / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < BLOCK / 32) sh[lane] = s;
  }
  __syncthreads();
  const int base = wid ? sh[wid - 1] : 0;
  total = sh[BLOCK / 32 - 1];
  __syncthreads();
  return base + x - v;
}

#ifdef LM_DIAG
// diagnostics build only (-DLM_DIAG): per apply-round maximum of each phase's per-thread
// elapsed time, summed over rounds (g_diag[8 + phase]); g_diag[0..7] per-round scratch
__device__ unsigned long long g_diag[64];
__device__ __forceinline__ void diag_fold(int bank) {  // per-round maxima of one bank -> sums
  for (int ph = 0; ph < 5; ++ph) {
    g_diag[8 + ph] += g_diag[5 * bank + ph + 32];
    g_diag[5 * bank + ph + 32] = 0;
  }
  g_diag[16] += 1;
}
__device__ __forceinline__ void diag_max(int phase, long long t_start) {
  unsigned long long e = (unsigned long long)(gtime() - t_start);
  for (int off = 16; off; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(__activemask(), e, off);
    e = o > e ? o : e;
  }
  atomicMax(&g_diag[phase + 32], e);
}
#define DIAG_T0 long long diag_t0 = gtime();
#define DIAG_RESTART diag_t0 = gtime();
#define DIAG_MAX(ph) if (Team::kCluster) diag_max(ph + 5 * (rounds & 1), diag_t0);
#else
#define DIAG_T0
#define DIAG_RESTART
#define DIAG_MAX(ph)
#endif

// warp-aggregated atomicAdd(p, 1) over the threads active here: one atomic per warp (the
// team control words live in one CTA's shared memory and every CTA of a cluster hits them)
__device__ __forceinline__ int agg_inc(int* p) {
  const unsigned am = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(p, __popc(am));
  base = __shfl_sync(am, base, leader);
  return base + __popc(am & ((1u << lane) - 1));
}

template <int BLOCK>
__device__ __forceinline__ int block_sum(int v, int* sh) {
  int t;
  block_excl_scan<BLOCK>(v, sh, t);
  return t;
}

__device__ __forceinline__ long long payload_bytes(const DevMap& M, int slot) {
  return (long long)M.kp_n[slot] * (M.kp_rec_bytes + M.desc_bytes);
}

// rank key of a covisibility entry: weight descending, then keyframe id ascending
__device__ __forceinline__ unsigned long long covis_key(const DevMap& M, int slot, int w) {
  return ((unsigned long long)(0x7fffffff - w) << 32) | (unsigned)M.kf_id[slot];
}

// covisible_neighbors(k, n) (mapmodel.py:269-273 + CovisibilityGraph.neighbors 100-105):
// live slots with weight >= min_w, ordered by (-weight, kf_id). Block-cooperative:
// compacts the row into shared (slot, key) pairs, ranks each entry by counting smaller
// keys and scatters to out[rank]; returns min(count, n) (n < 0: all).
template <int BLOCK>
__device__ int ranked_neighbors(const DevMap& M, int k, int n, int* sh_slot, unsigned long long* sh_key, int* out,
                                int n_slots) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int* row = M.covis + (size_t)k * M.kf_cap;
  for (int s = threadIdx.x; s < n_slots; s += BLOCK) {
    const int w = __ldcg(row + s);  // (L2: the row may change between kernels that run early under PDL)
    if (w >= M.min_w && w > 0 && s != k && M.kf_state[s] == KF_LIVE) {
      const int at = atomicAdd(&cnt, 1);
      sh_slot[at] = s;
      sh_key[at] = covis_key(M, s, w);
    }
  }
  __syncthreads();
  const int c = cnt;
  const int lim = n < 0 ? c : (n < c ? n : c);
  for (int e = threadIdx.x; e < c; e += BLOCK) {
    const unsigned long long ke = sh_key[e];
    int r = 0;
    for (int f = 0; f < c; ++f) r += sh_key[f] < ke;
    if (r < lim) out[r] = sh_slot[e];
  }
  __syncthreads();
  return lim;
}

// ---------------------------------------------------------------------------------- insert

__global__ void __launch_bounds__(256) k_insert(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.x];
  const DevMap& M = maps[A.map];
  {  // the step's statistics record starts from zero (16-byte stores; the record is 8-aligned)
    static_assert(sizeof(lm_step_stats) % 8 == 0, "stats record layout");
    long long* p = (long long*)M.s.stats;
    for (int k = threadIdx.x; k < (int)(sizeof(lm_step_stats) / 8); k += blockDim.x) p[k] = 0;
    if (threadIdx.x == 0) M.scal[SC_SOFT] = 0;
  }
  // (no barrier needed: thread 0 below writes none of the zeroed words; the kernel boundary
  // orders the zeroing before every later stage)
  if (!A.do_insert || threadIdx.x) return;
  const int slot = A.cur;
  const int off = M.kp_off[slot], n = M.kp_n[slot];
  const bool any = A.prebound != 0;  // staged with pre-bound slots (host-side flag)
  M.kf_state[slot] = KF_LIVE;
  if (A.do_upload) {  // upload_keyframe devicestore.py:68-78
    M.kf_res[slot] = 1;
    M.ledger[LG_PERSIST] += (unsigned long long)payload_bytes(M, slot);
  }
  if (!any) return;
  // pre-bound slots register their observations in keypoint order (insert_keyframe
  // mapmodel.py:185-199); rare (tests, externally seeded maps), so one thread
  for (int i = 0; i < n; ++i) {
    const int mp = M.kbind[off + i];
    if (mp < 0) continue;
    M.kbind[off + i] = -1;
    if (mp >= M.scal[SC_NEXT_ID] || !M.alive[mp] || obs_find(M, mp, slot) >= 0) {
      set_err(M, LM_ERR_INVALID_ARGUMENT);
      continue;
    }
    link(M, mp, slot, i);
    mark_dirty(M, mp);
  }
}

// ---------------------------------------------------------------------------------- cull

constexpr int CULL_CHUNK = 2048;  // probation entries per k_cull iteration (two per thread)
constexpr int CULL_DYN_SMEM = (3 * CULL_CHUNK + PAIR_W * (CULL_CHUNK / 32)) * 4;  // kill rows + transposed columns

template <bool P>
__global__ void __launch_bounds__(1024) k_cull(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  // one cluster per map: rank 0 classifies and owns the accumulator; every rank takes a share
  // of the kills' scattered record updates (one SM's load/store pipe was their bound)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), nranks = (int)cl.num_blocks();
  const StepArgs& A = args[blockIdx.x / nranks];
  const DevMap& M = maps[A.map];
  if (!A.do_cull) return;  // (uniform over the cluster)
  __shared__ int sh[32];
  __shared__ PairAcc acc;
  __shared__ int kills[CULL_CHUNK], big[CULL_CHUNK];
  __shared__ int nbig, nact_sh;
  extern __shared__ unsigned cull_dyn[];
  unsigned* krow = cull_dyn;                   // [3*CULL_CHUNK] per kill: observer window mask
  unsigned* kcol = cull_dyn + 3 * CULL_CHUNK;  // [CULL_CHUNK/32][PAIR_W] per window slot: mask over the kills
  __shared__ int kact[PAIR_W], kidx[PAIR_W];
  __shared__ int tk_sh;
  constexpr int CULL_HEAVY = 256;        // high-degree kills of this CTA handled warp-wide
  __shared__ int heavy[CULL_HEAVY], nheavy;
  int* kills0 = cl.map_shared_rank(kills, 0);
  int* big0 = cl.map_shared_rank(big, 0);
  int* nbig0 = cl.map_shared_rank(&nbig, 0);
  unsigned* krow0 = cl.map_shared_rank(krow, 0);
  const int* tk0 = cl.map_shared_rank(&tk_sh, 0);
  const long long c_t0 = gtime_p<P>();
  pair_acc_init<1024>(&acc, A.cur);
  const long long c_t1 = gtime_p<P>();
  long long c_kill = 0;
  const int n = M.scal[SC_RECENT_N];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int kept = 0, culled = 0, nbig_total = 0;
  for (int base = 0; base < n; base += CULL_CHUNK) {
    int tk = 0;
    if (rank == 0) {
    // two consecutive entries per thread (order-stable compaction)
    int keep[2] = {0, 0}, kill[2] = {0, 0}, id[2] = {-1, -1}, born[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = base + 2 * threadIdx.x + h;
      if (e < n) {
        id[h] = M.recent_id[e];
        born[h] = M.recent_born[e];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = id[h];
      if (i >= 0 && M.alive[i]) {  // dead entries (merged away) just leave the list
        const double ratio = (double)M.found[i] / (double)(M.visible[i] > 1 ? M.visible[i] : 1);
        if (ratio < A.cc.found_ratio_min) kill[h] = 1;
        else if (A.processed - born[h] >= A.cc.probation_kfs) kill[h] = M.nobs[i] < A.cc.min_obs_graduate;
        else keep[h] = 1;
      }
    }
    const int ak = block_excl_scan<1024>(kill[0] + kill[1], sh, tk);
    if (kill[0]) kills[ak] = id[0];
    if (kill[1]) kills[ak + kill[0]] = id[1];
    int tot;
    const int at = block_excl_scan<1024>(keep[0] + keep[1], sh, tot);
    if (keep[0]) {  // stable in-place compaction: write index <= read index
      M.recent_id[kept + at] = id[0];
      M.recent_born[kept + at] = born[0];
    }
    if (keep[1]) {
      M.recent_id[kept + at + keep[0]] = id[1];
      M.recent_born[kept + at + keep[0]] = born[1];
    }
    kept += tot;
    culled += tk;
    if (threadIdx.x == 0) {
      nbig = 0;
      tk_sh = tk;
    }
    }
    cl.sync();  // the chunk's kill list (rank 0) is published
    const long long c_a = gtime_p<P>();
    // independent points, thread each, spread over the cluster: bindings and counters
    // cleared, the observer set as a window bitmask (rows, into rank 0); the covisibility
    // decrements of all of them are the pair counts of the rows' Gram matrix, counted with
    // popcounts over the transposed masks instead of one contended shared atomic per
    // observer pair. Kills with an observer outside the window take the per-pair path.
    tk = *tk0;
    // a kill's chain is ~3 dependent L2 round trips per 8 observations on one thread, so the
    // few long-lived probation points (tens of observations, most of them fusion ADDs) set the
    // phase's critical path: points with more than HEAVY observations go to a warp each (lanes
    // over the observations) after the thread pass
    constexpr int HEAVY = 16;
    if (threadIdx.x == 0) nheavy = 0;
    __syncthreads();
    for (int k = rank + nranks * threadIdx.x; k < tk; k += nranks * 1024) {
      const int id = kills0[k];
      if (M.nobs[id] > HEAVY) {
        const int at = atomicAdd(&nheavy, 1);
        if (at < CULL_HEAVY) {
          heavy[at] = k;
          continue;
        }
      }
      unsigned r[3];
      if (!kill_point_rows_thread(M, id, &acc, r)) {
        r[0] = r[1] = r[2] = 0u;
        big0[atomicAdd(nbig0, 1)] = id;
      }
      krow0[3 * k] = r[0];
      krow0[3 * k + 1] = r[1];
      krow0[3 * k + 2] = r[2];
    }
    __syncthreads();
    {
      const int nh = nheavy < CULL_HEAVY ? nheavy : CULL_HEAVY;
      for (int h = wid; h < nh; h += 32) {
        const int k = heavy[h];
        const int id = kills0[k];
        unsigned r[3] = {0u, 0u, 0u};
        if (!kill_point_rows_warp(M, id, lane, &acc, r)) {
          if (lane == 0) big0[atomicAdd(nbig0, 1)] = id;
          r[0] = r[1] = r[2] = 0u;
        }
        if (lane == 0) {
          krow0[3 * k] = r[0];
          krow0[3 * k + 1] = r[1];
          krow0[3 * k + 2] = r[2];
        }
      }
    }
    cl.sync();  // rows complete; ranks > 0 go on to the next chunk
    if (rank != 0) continue;
    for (int k = wid; k < nbig; k += 32) kill_point_warp(M, big[k], lane, &acc);  // outside the window
    nbig_total += nbig;
    {
      // transpose: column mask of window slot a over the kills (warp w: kills 32w..32w+31)
      const int nkw = (tk + 31) >> 5;
      for (int w = wid; w < nkw; w += 32) {
        const int k = 32 * w + lane;
        const unsigned r0 = k < tk ? krow[3 * k] : 0u, r1 = k < tk ? krow[3 * k + 1] : 0u;
        const unsigned r2 = k < tk ? krow[3 * k + 2] : 0u;
        for (int a = 0; a < PAIR_W; ++a) {
          const unsigned bit = a < 32 ? (r0 >> a) & 1u : a < 64 ? (r1 >> (a - 32)) & 1u : (r2 >> (a - 64)) & 1u;
          const unsigned col = __ballot_sync(0xffffffffu, bit);
          if (lane == 0) kcol[w * PAIR_W + a] = col;
        }
      }
      __syncthreads();
      // slots with any killed observer, then their pairs
      unsigned abal = 0u;
      if (wid < PAIR_W / 32) {
        unsigned any = 0u;
        for (int w = 0; w < nkw; ++w) any |= kcol[w * PAIR_W + threadIdx.x];
        abal = __ballot_sync(0xffffffffu, any != 0u);
        if (lane == 0) kact[wid] = __popc(abal);
      }
      __syncthreads();
      if (wid < PAIR_W / 32) {  // active slots in order
        int off = 0;
        for (int w = 0; w < wid; ++w) off += kact[w];
        if (abal >> lane & 1u) kidx[off + __popc(abal & ((1u << lane) - 1))] = threadIdx.x;
        if (threadIdx.x == 0) {
          int m = 0;
          for (int w = 0; w < PAIR_W / 32; ++w) m += kact[w];
          nact_sh = m;
        }
      }
      __syncthreads();
      const int m = nact_sh, np = m * (m - 1) / 2;
      for (int q = threadIdx.x; q < np; q += 1024) {
        int i = 0, rem = q;  // q -> (i < j) over the active slots
        while (rem >= m - 1 - i) {
          rem -= m - 1 - i;
          ++i;
        }
        const int a = kidx[i], b = kidx[i + 1 + rem];
        int c = 0;
        for (int w = 0; w < nkw; ++w) c += __popc(kcol[w * PAIR_W + a] & kcol[w * PAIR_W + b]);
        if (c) atomicAdd(&acc.win[tri_index(a, b)], -c);
      }
    }
    __syncthreads();
    c_kill += gtime_p<P>() - c_a;
  }
  if (rank != 0) return;
  const long long c_t2 = gtime_p<P>();
  pair_acc_flush<1024>(M, &acc);
  const long long c_t3 = gtime_p<P>();
  if (threadIdx.x == 0) {
    M.scal[SC_RECENT_N] = kept;
    M.s.stats->culled = culled;
    M.s.stats->dbg[13] += n;  // diagnostics: probation list length
    M.s.stats->dbg[14] += nbig_total;
    M.s.stats->dbg[1] += c_t1 - c_t0;            // cull: accumulator init (ns)
    M.s.stats->dbg[1] += c_t2 - c_t1 - c_kill;   // cull: init + classification + compaction
    M.s.stats->dbg[2] += c_kill;                 // cull: kills
    M.s.stats->dbg[3] += c_t3 - c_t2;            // cull: covisibility flush
  }
}

// ---------------------------------------------------------------------------------- select

__device__ __forceinline__ void k_select_body(DevMap* maps, const StepArgs* args, int n_slots_max) {
  const StepArgs& A = args[blockIdx.x];
  const DevMap& M = maps[A.map];
  if (!A.do_create) return;
  extern __shared__ unsigned long long dynk[];
  unsigned long long* sh_key = dynk;
  int* sh_slot = (int*)(dynk + M.kf_cap);
  __shared__ int out[NMAX];
  __shared__ int n_out;
  const int cur = A.cur;
  int want = A.n_nbr_req < NMAX ? A.n_nbr_req : NMAX;
  if (A.explicit_nbr) {
    if (threadIdx.x == 0) {
      out[0] = A.nbr0;
      n_out = 1;
    }
    __syncthreads();
  } else {
    const int got = ranked_neighbors<256>(M, cur, want, sh_slot, sh_key, out, n_slots_max);
    if (threadIdx.x == 0) n_out = got;
    __syncthreads();
    if (n_out < want) {
      // recency padding: live keyframes other than cur, newest kf id first, not yet listed
      __shared__ int cnt;
      if (threadIdx.x == 0) cnt = 0;
      __syncthreads();
      for (int s = threadIdx.x; s < n_slots_max; s += 256) {
        if (s == cur || M.kf_state[s] != KF_LIVE) continue;
        bool listed = false;
        for (int k = 0; k < n_out; ++k) listed |= out[k] == s;
        if (!listed) sh_slot[atomicAdd(&cnt, 1)] = s;
      }
      __syncthreads();
      const int c = cnt, need = want - n_out;
      for (int e = threadIdx.x; e < c; e += 256) {
        const long long ie = M.kf_id[sh_slot[e]];
        int r = 0;
        for (int f = 0; f < c; ++f) r += M.kf_id[sh_slot[f]] > ie;
        if (r < need) out[n_out + r] = sh_slot[e];
      }
      __syncthreads();
      if (threadIdx.x == 0) n_out = n_out + (c < need ? c : need);
      __syncthreads();
    }
  }
  // record_neighbor_access (devicestore.py:80-92): every neighbour must be resident, else
  // the stage fails before touching the map (InvalidStateError in the reference)
  const bool nonres = __syncthreads_or(threadIdx.x < n_out && !A.explicit_nbr && !M.scal[SC_NORES] &&
                                       !M.kf_res[out[threadIdx.x]]);
  if (nonres && threadIdx.x == 0) atomicCAS(&M.scal[SC_SOFT], 0, LM_ERR_INVALID_STATE);
  const int nn = nonres ? 0 : n_out;
  lm_step_stats* st = M.s.stats;
  if (threadIdx.x < nn) {
    const int s = out[threadIdx.x];
    M.s.nbr[threadIdx.x] = s;
    double F[9];
    const double ca[4] = {M.cam[6 * cur], M.cam[6 * cur + 1], M.cam[6 * cur + 2], M.cam[6 * cur + 3]};
    const double cb[4] = {M.cam[6 * s], M.cam[6 * s + 1], M.cam[6 * s + 2], M.cam[6 * s + 3]};
    const bool ok = fundamental(M.q + 4 * cur, M.t + 3 * cur, M.q + 4 * s, M.t + 3 * s, ca, cb, F);
    M.s.deg[threadIdx.x] = ok ? 0 : 1;
    for (int k = 0; k < 9; ++k) M.s.F[9 * threadIdx.x + k] = F[k];
    st->neighbors[threadIdx.x] = M.kf_id[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->n_neighbors = nn;
    int nd = 0;
    unsigned long long naive = 0;
    for (int r = 0; r < nn; ++r) {
      naive += (unsigned long long)payload_bytes(M, out[r]);
      if (M.s.deg[r]) st->degenerate_neighbors[nd++] = M.kf_id[out[r]];
    }
    st->n_degenerate_neighbors = nd;
    if (!A.explicit_nbr) M.ledger[LG_NAIVE] += naive;
  }
}

// With select_early (a freshly inserted keyframe without pre-bound slots: its covisibility
// row is empty, so the ranking reads nothing the recent-point cull writes) this kernel runs
// concurrently with k_cull: it lets its successor launch at once and waits for its
// predecessor (k_cull) only at the very end, so its own completion still implies k_cull's
// and the launch chain stays ordered.
__global__ void __launch_bounds__(256) k_select(DevMap* maps, const StepArgs* args, int n_slots_max) {
  const bool early = args[blockIdx.x].select_early != 0;
  if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  else pdl_enter();
  k_select_body(maps, args, n_slots_max);
  if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
}


// ---------------------------------------------------------------------------------- prep

__device__ __forceinline__ bool is_unbound(const DevMap& M, const StepArgs& A, int g, int local, bool cur_side) {
  if (cur_side ? A.use_mask_cur : A.use_mask_nbr) return (cur_side ? M.s.mask_cur : M.s.mask_nbr)[local] != 0;
  return M.kbind[g] < 0;
}

__global__ void __launch_bounds__(256) k_prep(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_create) return;
  const int nn = M.s.stats->n_neighbors;
  const int list = blockIdx.x;  // 0 = current, r+1 = neighbour r
  if (list > nn) return;
  __shared__ int lcount[LMAX], lstart[LMAX + 1], lcur[LMAX];
  const int L = M.L;
  const int slot = list == 0 ? A.cur : M.s.nbr[list - 1];
  const int r = list - 1;
  const int off = M.kp_off[slot], n = M.kp_n[slot];
  const int ncur = M.kp_n[A.cur];
  if (list > 0 && M.s.deg[r]) {
    if (threadIdx.x == 0) {
      M.s.nb_n[r] = 0;
      M.s.cand_n[r] = 0;
    }
    return;
  }
  if (threadIdx.x < LMAX) lcount[threadIdx.x] = 0;
  __syncthreads();
  // each thread's keypoints (i = tid + 256 q): unbound flag and level loaded in one round (the
  // per-keypoint shared atomics would otherwise put one L2 round trip per iteration on the chain)
  constexpr int PQ = 8;
  unsigned char lv[PQ];
  unsigned ub = 0u;
  const bool fits = n <= 256 * PQ;
  if (fits) {
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
      const int i = threadIdx.x + 256 * q;
      lv[q] = i < n ? M.klev[off + i] : 0;
      if (i < n && is_unbound(M, A, off + i, i, list == 0)) ub |= 1u << q;
    }
#pragma unroll
    for (int q = 0; q < PQ; ++q)
      if (ub >> q & 1u) atomicAdd(&lcount[lv[q]], 1);
  } else {
    for (int i = threadIdx.x; i < n; i += 256)
      if (is_unbound(M, A, off + i, i, list == 0)) atomicAdd(&lcount[M.klev[off + i]], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int l = 0; l < L; ++l) {
      lstart[l] = acc;
      lcur[l] = acc;
      acc += lcount[l];
    }
    lstart[L] = acc;
  }
  __syncthreads();
  if (list == 0) {
    if (fits) {
#pragma unroll
      for (int q = 0; q < PQ; ++q) {
        const int i = threadIdx.x + 256 * q;
        if (i < n) M.s.win_rank[i] = 0x7fffffff;
        if (ub >> q & 1u) M.s.cur_sorted[atomicAdd(&lcur[lv[q]], 1)] = i;
      }
    } else {
      for (int i = threadIdx.x; i < n; i += 256) {
        M.s.win_rank[i] = 0x7fffffff;
        if (is_unbound(M, A, off + i, i, true)) {
          const int at = atomicAdd(&lcur[M.klev[off + i]], 1);
          M.s.cur_sorted[at] = i;
        }
      }
    }
    if (threadIdx.x <= L) M.s.cur_bucket[threadIdx.x] = lstart[threadIdx.x];
    // tiles never straddle a level; they are listed longest first (k_match dispatches tiles
    // in this order, every neighbour's copy of a tile side by side), so the tail of the
    // wave is made of short tiles. Work proxy: tile size x the current keyframe's unbound
    // population of the tile's level window. Rank sort in shared memory.
    constexpr int TCAP = 512;
    __shared__ int t_l[TCAP], t_s[TCAP], t_c[TCAP], t_w[TCAP];
    __shared__ int nt_sh;
    if (threadIdx.x == 0) {
      int nt = 0;
      const int w = A.mc.level_window;
      for (int l = 0; l < L; ++l) {
        int win = 0;
        for (int q = l - w; q <= l + w; ++q)
          if (q >= 0 && q < L) win += lcount[q];
        for (int s = lstart[l]; s < lstart[l + 1]; s += MATCH_TILE) {
          const int c = lstart[l + 1] - s < MATCH_TILE ? lstart[l + 1] - s : MATCH_TILE;
          if (nt < TCAP) {
            t_l[nt] = l;
            t_s[nt] = s;
            t_c[nt] = c;
            t_w[nt] = c * win;
          } else {
            M.s.tiles[3 * nt] = l;  // (beyond the sort capacity: appended unsorted)
            M.s.tiles[3 * nt + 1] = s;
            M.s.tiles[3 * nt + 2] = c;
          }
          ++nt;
        }
      }
      nt_sh = nt;
      *M.s.n_tiles = nt;
    }
    __syncthreads();
    const int ns = nt_sh < TCAP ? nt_sh : TCAP;
    for (int a = threadIdx.x; a < ns; a += 256) {
      int rk = 0;
      for (int b = 0; b < ns; ++b) rk += t_w[b] > t_w[a] || (t_w[b] == t_w[a] && b < a);
      M.s.tiles[3 * rk] = t_l[a];
      M.s.tiles[3 * rk + 1] = t_s[a];
      M.s.tiles[3 * rk + 2] = t_c[a];
    }
  } else {
    const size_t base = (size_t)r * M.kpkf_max;
    auto put = [&](int i, int lvi) {  // (the copies' loads issue before the slot atomic)
      const uint4 d0 = M.kdesc[2 * (off + i)], d1 = M.kdesc[2 * (off + i) + 1];
      const double u = M.ku[off + i], v = M.kv[off + i];
      const int at = atomicAdd(&lcur[lvi], 1);
      M.s.nb_j[base + at] = i;
      M.s.nb_desc[2 * (base + at)] = d0;
      M.s.nb_desc[2 * (base + at) + 1] = d1;
      M.s.nb_u[base + at] = u;
      M.s.nb_v[base + at] = v;
      M.s.nb_thr[base + at] = A.mc.chi2_epi * M.S2[lvi];
    };
    if (fits) {
#pragma unroll
      for (int q = 0; q < PQ; ++q) {
        const int i = threadIdx.x + 256 * q;
        if (i < n) M.s.bestj[base + i] = ~0ull;
        if (ub >> q & 1u) put(i, lv[q]);
      }
    } else {
      for (int i = threadIdx.x; i < n; i += 256) {
        M.s.bestj[base + i] = ~0ull;
        if (is_unbound(M, A, off + i, i, false)) put(i, M.klev[off + i]);
      }
    }
    for (int i = threadIdx.x; i < ncur; i += 256) M.s.pick[base + i] = ~0ull;
    if (threadIdx.x <= L) M.s.nb_bucket[r * (LMAX + 1) + threadIdx.x] = lstart[threadIdx.x];
    if (threadIdx.x == 0) M.s.nb_n[r] = lstart[L];
  }
}

// ---------------------------------------------------------------------------------- match

// grid (tiles, NMAX, maps), block MATCH_WARPS x 32. A tile is 32 unbound current keypoints
// of one pyramid level (lane = keypoint); the CTA's warps split the neighbour's unbound
// keypoints of levels [l-w, l+w] (contiguous in the level-bucketed list) into slices.
// Descriptors are staged in shared memory and read warp-uniformly (broadcast). Hamming
// first: the 128-bit prefix distance already exceeds the limit for almost every
// non-matching pair, so the second half and the fp64 epipolar test run only on survivors.
// The running minimum is the lexicographic (dist, j) key of the reference's first-argmin;
// warp slices combine with a shared atomicMin, neighbour one-to-one with a global one.
__global__ void __launch_bounds__(MATCH_WARPS * 32, 5) k_match(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  if (!A.do_create) return;
  const int r = blockIdx.x;  // neighbour fastest: each tile's copies dispatch side by side
  if (r >= M.s.stats->n_neighbors || M.s.deg[r]) return;
  const int tile = blockIdx.y;
  if (tile >= *M.s.n_tiles) return;
  __shared__ uint4 sd[2 * MATCH_JT];
  __shared__ unsigned long long best_sh[MATCH_TILE];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int lv = M.s.tiles[3 * tile], start = M.s.tiles[3 * tile + 1], cnt = M.s.tiles[3 * tile + 2];
  const int w = A.mc.level_window;
  const int l0 = lv - w < 0 ? 0 : lv - w;
  const int l1 = lv + w > M.L - 1 ? M.L - 1 : lv + w;
  const int* bk = M.s.nb_bucket + r * (LMAX + 1);
  const int jb = bk[l0], je = bk[l1 + 1];
  const size_t base = (size_t)r * M.kpkf_max;
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)&M.s.stats->match_pairs, (unsigned long long)cnt * (je - jb));
  if (threadIdx.x < MATCH_TILE) best_sh[threadIdx.x] = ~0ull;
  const int cur = A.cur;
  const int off = M.kp_off[cur];
  const bool active = lane < cnt;
  int i = 0;
  uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0;
  double l[3] = {0, 0, 0}, den = 0;
  if (active) {
    i = M.s.cur_sorted[start + lane];
    a0 = M.kdesc[2 * (off + i)];
    a1 = M.kdesc[2 * (off + i) + 1];
    epi_line(M.s.F + 9 * r, M.ku[off + i], M.kv[off + i], l);
    den = l[0] * l[0] + l[1] * l[1];
  }
  const int maxd = A.mc.match_max_distance;
  unsigned long long best = ~0ull;
  int border = 0, second = 0;
  for (int c0 = jb; c0 < je; c0 += MATCH_JT) {
    const int cn = je - c0 < MATCH_JT ? je - c0 : MATCH_JT;
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * cn; k += MATCH_WARPS * 32) sd[k] = M.s.nb_desc[2 * (base + c0) + k];
    __syncthreads();
    // this warp's slice of the chunk
    const int per = (cn + MATCH_WARPS - 1) / MATCH_WARPS;
    const int k0 = wid * per, k1 = k0 + per < cn ? k0 + per : cn;
    if (active) {
#pragma unroll 2
      for (int k = k0; k < k1; ++k) {
        const uint4 b0 = sd[2 * k];
        int dist = __popc(a0.x ^ b0.x) + __popc(a0.y ^ b0.y) + __popc(a0.z ^ b0.z) + __popc(a0.w ^ b0.w);
        if (dist <= maxd) {
          ++second;
          const uint4 b1 = sd[2 * k + 1];
          dist += __popc(a1.x ^ b1.x) + __popc(a1.y ^ b1.y) + __popc(a1.z ^ b1.z) + __popc(a1.w ^ b1.w);
          if (dist <= maxd) {
            const size_t e = base + c0 + k;
            const double d2 = epi_d2(l, den, M.s.nb_u[e], M.s.nb_v[e]), thr = M.s.nb_thr[e];
            border += near_tie(d2, thr, thr);
            if (d2 <= thr) {
              const unsigned long long key = ((unsigned long long)dist << 32) | (unsigned)M.s.nb_j[e];
              best = key < best ? key : best;
            }
          }
        }
      }
    }
  }
  if (active && best != ~0ull) atomicMin(&best_sh[lane], best);
  if (__any_sync(0xffffffffu, border)) {
    for (int o = 16; o; o >>= 1) border += __shfl_xor_sync(0xffffffffu, border, o);
    if (lane == 0) atomicAdd((unsigned long long*)&M.s.stats->borderline[0], (unsigned long long)border);
  }
  {  // executed-popcount diagnostic: one same-address atomic per CTA, not per warp
    __shared__ int sec_sh;
    if (threadIdx.x == 0) sec_sh = 0;
    for (int o = 16; o; o >>= 1) second += __shfl_xor_sync(0xffffffffu, second, o);
    __syncthreads();
    if (lane == 0 && second) atomicAdd(&sec_sh, second);
    __syncthreads();
    if (threadIdx.x == 0 && sec_sh)
      atomicAdd((unsigned long long*)&M.s.stats->match_second_half, (unsigned long long)sec_sh);
  }
  __syncthreads();
  if (wid == 0 && active) {
    const unsigned long long b = best_sh[lane];
    M.s.pick[base + i] = b;
    if (b != ~0ull) {
      const unsigned j = (unsigned)(b & 0xffffffffu);
      atomicMin(&M.s.bestj[base + j], (b & 0xffffffff00000000ull) | (unsigned)i);
    }
  }
}

// ---------------------------------------------------------------------------------- tri

// grid (neighbour, slice, map): every slice CTA of a neighbour compacts the one-to-one
// survivors (cheap: two rounds of L2 loads per thread) into its shared memory and takes every
// gridDim.y-th of them, so the fp64 triangulations (one Jacobi SVD per thread, the kernel's
// critical path) spread over gridDim.y SMs; slice 0 also writes the compacted list for
// k_commit. Without shared memory (dynamic size 0: very large keyframes) one slice reads the
// list back from global memory.
__global__ void __launch_bounds__(256) k_tri(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  if (!A.do_create) return;
  const int r = blockIdx.x;
  const int slice = blockIdx.y, nslice = gridDim.y;
  if (r >= M.s.stats->n_neighbors) return;
  if (M.s.deg[r]) return;  // cand_n[r] = 0 set by k_prep
  if (slice > 0 && A.search_only) return;
  extern __shared__ int tri_sm[];  // [kpkf_max] current index, [kpkf_max] neighbour index
  const bool use_sm = dyn_smem_bytes() >= 8u * (unsigned)M.kpkf_max;
  __shared__ int sh[32];
  const int cur = A.cur;
  const int ncur = M.kp_n[cur];
  const size_t base = (size_t)r * M.kpkf_max;
  // one-to-one survivors in current-index order: each thread owns TQ consecutive keypoints
  // (all their pick / bestj loads in two rounds), one block scan per 256 * TQ keypoints
  constexpr int TQ = 8;
  int count = 0;
  for (int b0 = 0; b0 < ncur; b0 += 256 * TQ) {
    const int i0 = b0 + threadIdx.x * TQ;
    unsigned long long pk[TQ], bj[TQ];
#pragma unroll
    for (int q = 0; q < TQ; ++q) pk[q] = i0 + q < ncur ? M.s.pick[base + i0 + q] : ~0ull;
#pragma unroll
    for (int q = 0; q < TQ; ++q) bj[q] = pk[q] != ~0ull ? M.s.bestj[base + (unsigned)(pk[q] & 0xffffffffu)] : 0ull;
    unsigned fl = 0u;
#pragma unroll
    for (int q = 0; q < TQ; ++q)
      if (pk[q] != ~0ull && bj[q] == ((pk[q] & 0xffffffff00000000ull) | (unsigned)(i0 + q))) fl |= 1u << q;
    int tot;
    int at = block_excl_scan<256>(__popc(fl), sh, tot);
#pragma unroll
    for (int q = 0; q < TQ; ++q)
      if (fl >> q & 1u) {
        const int k = count + at;
        if (use_sm) {
          tri_sm[k] = i0 + q;
          tri_sm[M.kpkf_max + k] = (int)(pk[q] & 0xffffffffu);
        }
        if (slice == 0) {
          M.s.cand_i[base + k] = i0 + q;
          M.s.cand_j[base + k] = (int)(pk[q] & 0xffffffffu);
          M.s.cand_d[base + k] = (int)(pk[q] >> 32);
        }
        ++at;
      }
    count += tot;
  }
  // the triangulation loop below reads candidate records other threads just wrote (shared or
  // global memory: they are visible block-wide only after a barrier)
  __syncthreads();
  if (threadIdx.x == 0 && slice == 0) M.s.cand_n[r] = count;
  if (A.search_only) return;
  if (!use_sm && slice > 0) return;  // (launched with one slice then)
  const int nb = M.s.nbr[r];
  const int offa = M.kp_off[cur], offb = M.kp_off[nb];
  for (int k = slice + nslice * threadIdx.x; k < count; k += 256 * nslice) {
    const int i = use_sm ? tri_sm[k] : M.s.cand_i[base + k];
    const int j = use_sm ? tri_sm[M.kpkf_max + k] : M.s.cand_j[base + k];
    const int ga = offa + i, gb = offb + j;
    double X[3] = {0, 0, 0};
    int st, border = 0;
    if (!triangulate(M.P + 12 * cur, M.P + 12 * nb, M.C + 3 * cur, M.C + 3 * nb, M.ku[ga], M.kv[ga], M.ku[gb],
                     M.kv[gb], X, &border)) {
      st = CS_DEGEN;
    } else {
      const int la = M.klev[ga], lb = M.klev[gb];
      ViewGeo va{M.R + 9 * cur, M.t + 3 * cur, M.C + 3 * cur, M.cam[6 * cur], M.cam[6 * cur + 1],
                 M.cam[6 * cur + 2], M.cam[6 * cur + 3], M.ku[ga], M.kv[ga], M.S2[la], M.S[la], M.sf};
      ViewGeo vb{M.R + 9 * nb, M.t + 3 * nb, M.C + 3 * nb, M.cam[6 * nb], M.cam[6 * nb + 1],
                 M.cam[6 * nb + 2], M.cam[6 * nb + 3], M.ku[gb], M.kv[gb], M.S2[lb], M.S[lb], M.sf};
      st = creation_gates(va, vb, X, A.gc.cos_parallax_max, A.gc.chi2_mono, A.gc.scale_ratio_slack, &border);
    }
    if (border) atomicAdd((unsigned long long*)&M.s.stats->borderline[1], (unsigned long long)border);
    M.s.cand_st[base + k] = st;
    M.s.cand_X[3 * (base + k)] = X[0];
    M.s.cand_X[3 * (base + k) + 1] = X[1];
    M.s.cand_X[3 * (base + k) + 2] = X[2];
    if (st == CS_PASS) atomicMin(&M.s.win_rank[i], r);
  }
}

// ---------------------------------------------------------------------------------- commit

__global__ void __launch_bounds__(1024) k_commit(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.x];
  const DevMap& M = maps[A.map];
  if (!A.do_create || A.search_only) return;
  __shared__ int sh[32];
  __shared__ int coff[NMAX + 1];
  __shared__ int per_r[NMAX];
  __shared__ int okcap;
  const int nn = M.s.stats->n_neighbors;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int r = 0; r < nn; ++r) {
      coff[r] = acc;
      acc += M.s.cand_n[r];
    }
    coff[nn] = acc;
  }
  if (threadIdx.x < NMAX) per_r[threadIdx.x] = 0;
  __syncthreads();
  const int total = coff[nn];
  const int cur = A.cur;
  // outcome of candidate g: 0 created, 1 conflict, 2+ failure status. Every thread's
  // candidates (g = tid + 1024 q) are classified once, their loads issued together, and kept
  // in registers for the ranking pass below (candidate totals beyond CQ*1024 fall back to
  // recomputing).
  constexpr int CQ = 8;
  auto locate = [&](int g, int& r, int& k) {
    int lo = 0, hi = nn;  // largest r with coff[r] <= g (binary search over <= 64 neighbours)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (coff[mid] <= g) lo = mid;
      else hi = mid;
    }
    r = lo;
    k = g - coff[r];
  };
  auto outcome = [&](int g, int& r, int& k) -> int {
    locate(g, r, k);
    const size_t e = (size_t)r * M.kpkf_max + k;
    const int i = M.s.cand_i[e];
    if (M.s.win_rank[i] < r) return 1;
    const int st = M.s.cand_st[e];
    return st == CS_PASS ? 0 : 1 + st;
  };
  int ocs[CQ], rs[CQ], ks[CQ];
  {
    int ci[CQ], cst[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int g = threadIdx.x + 1024 * q;
      rs[q] = ks[q] = 0;
      ci[q] = 0;
      cst[q] = 0;
      if (g < total) {
        locate(g, rs[q], ks[q]);
        const size_t e = (size_t)rs[q] * M.kpkf_max + ks[q];
        ci[q] = M.s.cand_i[e];
        cst[q] = M.s.cand_st[e];
      }
    }
    int wr[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) wr[q] = threadIdx.x + 1024 * q < total ? M.s.win_rank[ci[q]] : 0;
#pragma unroll
    for (int q = 0; q < CQ; ++q)
      ocs[q] = threadIdx.x + 1024 * q >= total ? -1 : (wr[q] < rs[q] ? 1 : (cst[q] == CS_PASS ? 0 : 1 + cst[q]));
  }
  // pass 1: totals and capacity (one combined block reduction)
  int cnt7[7] = {0, 0, 0, 0, 0, 0, 0};  // created, conflicts, degenerate, parallax, depth, reproj, scale
  auto tally = [&](int oc) {  // (constant indices only: the counters stay in registers)
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const int want = c == 0 ? 0 : c == 1 ? 1 : c == 2 ? 1 + CS_DEGEN : 1 + (c - 2);
      cnt7[c] += oc == want;
    }
  };
#pragma unroll
  for (int q = 0; q < CQ; ++q) tally(ocs[q]);
  for (int g = threadIdx.x + 1024 * CQ; g < total; g += 1024) {
    int r, k;
    tally(outcome(g, r, k));
  }
  __shared__ int red[32][7];
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      int v = cnt7[c];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wid][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
      int v = 0;
      for (int w = 0; w < 32; ++w) v += red[w][threadIdx.x];
      red[0][threadIdx.x] = v;  // (row 0 read back by thread threadIdx.x only, then synced)
    }
    __syncthreads();
  }
  const int created = red[0][0], conflicts = red[0][1], degen = red[0][2];
  int gates[4];
  for (int q = 0; q < 4; ++q) gates[q] = red[0][3 + q];
  const int id0 = M.scal[SC_NEXT_ID];
  const int obs0 = M.scal[SC_OBS_HEAD];
  const int rec0 = M.scal[SC_RECENT_N];
  if (threadIdx.x == 0) {
    okcap = 1;
    if ((long long)id0 + created > M.mp_cap || (long long)obs0 + 4LL * created > M.obs_cap ||
        rec0 + created > M.recent_cap) {
      okcap = 0;
      set_err(M, LM_ERR_CAPACITY);
    }
  }
  __syncthreads();
  // creation ranks (the records are written wide by k_commit_write: one SM's load/store
  // pipe bounds ~900 scattered record writes)
  if (threadIdx.x == 0) {
    M.s.cmeta[0] = id0;
    M.s.cmeta[1] = obs0;
    M.s.cmeta[2] = rec0;
  }
  {
    int run = 0;
    for (int b0 = 0, q = 0; b0 < total; b0 += 1024, ++q) {
      const int g = b0 + threadIdx.x;
      int r = 0, k = 0, oc = -1;
      if (q < CQ) {
#pragma unroll
        for (int u = 0; u < CQ; ++u)
          if (u == q) {
            oc = ocs[u];
            r = rs[u];
            k = ks[u];
          }
      } else if (g < total) {
        oc = outcome(g, r, k);
      }
      int tot;
      const int at = block_excl_scan<1024>(oc == 0, sh, tot);
      if (g < total) M.s.crank[(size_t)r * M.kpkf_max + k] = okcap && oc == 0 ? run + at : -1;
      if (okcap && oc == 0) atomicAdd(&per_r[r], 1);
      run += tot;
    }
  }
  __syncthreads();
  if (okcap && threadIdx.x < nn && per_r[threadIdx.x]) covis_add(M, cur, M.s.nbr[threadIdx.x], per_r[threadIdx.x]);
  if (threadIdx.x == 0) {
    lm_step_stats* st = M.s.stats;
    st->created = okcap ? created : 0;
    st->conflicts = conflicts;
    st->degenerate = degen;
    st->gate_parallax = gates[0];
    st->gate_depth = gates[1];
    st->gate_reprojection = gates[2];
    st->gate_scale = gates[3];
    st->first_new_id = id0;
    st->n_candidates = total;
    if (okcap) {
      M.scal[SC_NEXT_ID] = id0 + created;
      M.scal[SC_OBS_HEAD] = obs0 + 4 * created;
      M.scal[SC_RECENT_N] = rec0 + created;
    }
  }
}

// the new points' records, thread per (neighbour, candidate) of k_commit's ranks
__global__ void __launch_bounds__(128) k_commit_write(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  if (!A.do_create || A.search_only) return;
  const int r = blockIdx.y;
  if (r >= M.s.stats->n_neighbors) return;
  const int k = blockIdx.x * 128 + threadIdx.x;
  if (k >= M.s.cand_n[r]) return;
  const size_t e = (size_t)r * M.kpkf_max + k;
  const int rank = M.s.crank[e];
  if (rank < 0) return;
  const int cur = A.cur;
  const int id0 = M.s.cmeta[0], obs0 = M.s.cmeta[1], rec0 = M.s.cmeta[2];
  const int id = id0 + rank;
  const int i = M.s.cand_i[e], j = M.s.cand_j[e];
  const int nb = M.s.nbr[r];
  const int ga = M.kp_off[cur] + i, gb = M.kp_off[nb] + j;
  M.pos[3 * id] = M.s.cand_X[3 * e];
  M.pos[3 * id + 1] = M.s.cand_X[3 * e + 1];
  M.pos[3 * id + 2] = M.s.cand_X[3 * e + 2];
  const bool cur_first = M.kf_id[cur] < M.kf_id[nb];
  const int grep = cur_first ? ga : gb;
  M.rep[2 * id] = M.kdesc[2 * grep];
  M.rep[2 * id + 1] = M.kdesc[2 * grep + 1];
  M.alive[id] = 1;
  M.found[id] = 1;
  M.visible[id] = 1;
  M.first_kf[id] = M.kf_id[cur];
  const int oo = obs0 + 4 * rank;
  M.ooff[id] = oo;
  M.ocap[id] = 4;
  M.nobs[id] = 2;
  M.obs[oo] = cur_first ? make_int2(cur, i) : make_int2(nb, j);
  M.obs[oo + 1] = cur_first ? make_int2(nb, j) : make_int2(cur, i);
  M.dirty[id] = 0;
  M.gval[id] = 0;
  {  // a new point's counter row, written whole (no read-modify-write)
    const int la = M.klev[ga], lb = M.klev[gb];
    int* crow = M.counts + (size_t)id * M.L;
    for (int l = 0; l < M.L; ++l) crow[l] = (l == la) + (l == lb);
  }
  M.kbind[ga] = id;
  M.kbind[gb] = id;
  M.recent_id[rec0 + rank] = id;
  M.recent_born[rec0 + rank] = A.processed;
}

// ---------------------------------------------------------------------------------- fusion
//
// SearchAndFuse (fusion.py:307-347) for one keyframe, as a chain of kernels:
//   k_fuse_targets  1 CTA/map  collect_fusion_targets + forward point list + ledger
//   k_fuse_geo      warp/point refresh stale rep descriptors + view geometry of the forward points
//   k_fuse_gather   thread per (target, point): project, gate, window search, action build
//                   (all targets against the unchanged map, as the reference's gather-all)
//   k_fuse_apply    1 CTA/map  ordered apply of the forward batch (deterministic reservations)
//   k_fuse_refresh  warp/point refresh every point the forward apply touched
//   k_fuse_rev      1 CTA/map  reverse passes, gather -> apply per target (fusion.py:337-346)

// _point_geometry row (fusion.py:57-94) from the cached accumulators. Every field is
// loaded up front (one round of independent loads) before the validity branches.
__device__ void point_geometry(const DevMap& M, int mp, double slack, PGeo& g) {
  g.ok = 0;
  if (mp < 0) return;
  const bool alive = M.alive[mp] != 0;
  const int nobs = M.nobs[mp];
  const bool gv = M.gval[mp] != 0;
  double lo = M.glo[mp], hi = M.ghi[mp];
  double ax = M.gacc[3 * mp], ay = M.gacc[3 * mp + 1], az = M.gacc[3 * mp + 2];
  const double px = M.pos[3 * mp], py = M.pos[3 * mp + 1], pz = M.pos[3 * mp + 2];
  const uint4 r0 = M.rep[2 * mp], r1 = M.rep[2 * mp + 1];
  if (!alive || nobs == 0) return;
  if (!gv) {
    geo_full(M, mp);
    lo = M.glo[mp];
    hi = M.ghi[mp];
    ax = M.gacc[3 * mp];
    ay = M.gacc[3 * mp + 1];
    az = M.gacc[3 * mp + 2];
  }
  if (!isfinite(lo)) return;
  const double nrm = sqrt(ax * ax + ay * ay + az * az);
  if (nrm > 0) {
    g.vx = ax / nrm;
    g.vy = ay / nrm;
    g.vz = az / nrm;
  } else {
    g.vx = ax;
    g.vy = ay;
    g.vz = az;
  }
  g.x = px;
  g.y = py;
  g.z = pz;
  g.d0 = lo;
  g.blo = lo / slack;
  g.bhi = hi * M.S[M.L - 1] * slack;
  g.r0 = r0;
  g.r1 = r1;
  g.ok = 1;
}

// target keyframe's keypoints + cell grid, from global memory or a shared-memory copy
struct TgtView {
  const double* u;
  const double* v;
  const unsigned char* lev;
  const uint4* desc;
  const int* cst;    // cell starts [cells+1]
  const int* items;  // local keypoint index per cell entry
  const double* pose;  // R[9], t[3], C[3], cam[6], cell size
  int nx, ny;          // grid cells
};

__device__ __forceinline__ TgtView tgt_global(const DevMap& M, int ts) {
  const int off = M.kp_off[ts];
  return TgtView{M.ku + off, M.kv + off, M.klev + off, M.kdesc + 2 * (size_t)off,
                 M.cell_start + (size_t)ts * (GRID_CELLS + 1), M.cell_items + off, nullptr, M.g_nx[ts], M.g_ny[ts]};
}

// project + gates + grid window search for one (point, target) pair (fusion.py:97-129,
// 178-196). Returns -2 if the point is not visible in the target, -1 if visible without a
// hit, else the hit keypoint (lowest (distance, index) within the window).
// projection, gates and the conservative cell window of one (point, target) pair
struct GWin {
  double u, v, r2;
  int lp, x0, x1, y0, y1;
};

// border (optional): +1 to border[0] when the visibility decision rests on a borderline
// compare (no clearly failing one, at least one near_tie), +1 to border[1] for a rint tie of
// the predicted level
__device__ __forceinline__ bool gather_window(const DevMap& M, const lm_fuse_cfg& fc, const PGeo& g, int ts,
                                              const TgtView& T, GWin& w, int* border = nullptr) {
  if (!g.ok) return false;
  const double* R = T.pose ? T.pose : M.R + 9 * ts;
  const double* t = T.pose ? T.pose + 9 : M.t + 3 * ts;
  const double* C = T.pose ? T.pose + 12 : M.C + 3 * ts;
  const double* cam = T.pose ? T.pose + 15 : M.cam + 6 * ts;
  const double qx = R[0] * g.x + R[1] * g.y + R[2] * g.z;
  const double qy = R[3] * g.x + R[4] * g.y + R[5] * g.z;
  const double qz = R[6] * g.x + R[7] * g.y + R[8] * g.z;
  const double zc = qz + t[2];
  const double u = cam[0] * ((qx + t[0]) / zc) + cam[2];
  const double v = cam[1] * ((qy + t[1]) / zc) + cam[3];
  const bool inview = zc > 0 && u >= 0 && u < cam[4] && v >= 0 && v < cam[5];
  const double dx = g.x - C[0], dy = g.y - C[1], dz = g.z - C[2];
  const double d = sqrt(dx * dx + dy * dy + dz * dz);
  const double cosv = (dx * g.vx + dy * g.vy + dz * g.vz) / d;
  if (border) {
    const int near = near_tie(zc, 0.0, fabs(qz) + fabs(t[2])) + near_tie(u, 0.0, cam[4]) + near_tie(u, cam[4], cam[4]) +
                     near_tie(v, 0.0, cam[5]) + near_tie(v, cam[5], cam[5]) + near_tie(d, g.blo, d) +
                     near_tie(d, g.bhi, d) + near_tie(cosv, fc.min_view_cos, 1.0);
    if (near) {  // a clearly failing compare decides regardless of the borderline ones
      const double e = kFlipRel;
      const bool clear_fail = zc < -e * (fabs(qz) + fabs(t[2])) || u < -e * cam[4] || u > cam[4] * (1 + e) ||
                              v < -e * cam[5] || v > cam[5] * (1 + e) || d < g.blo - e * d || d > g.bhi + e * d ||
                              cosv < fc.min_view_cos - e;
      if (!clear_fail) border[0] += 1;
    }
  }
  if (!(zc > 0 && inview && d >= g.blo && d <= g.bhi)) return false;
  if (!(cosv >= fc.min_view_cos)) return false;
  double lraw = log(d / g.d0) / M.log_sf;
  if (!isfinite(lraw)) lraw = 0.0;
  if (border) border[1] += near_tie(lraw - floor(lraw), 0.5, lraw > 1.0 ? lraw : 1.0);
  double lr = rint(lraw);
  lr = lr < 0 ? 0 : (lr > M.L - 1 ? M.L - 1 : lr);
  w.lp = (int)lr;
  const double rad = fc.fuse_radius * M.S[w.lp];
  // conservative cell window, exact test inside
  const double cs = T.pose ? T.pose[21] : M.g_cs[ts];
  const int nx = T.nx, ny = T.ny;
  int x0 = (int)floor((u - rad - 1.0) / cs), x1 = (int)floor((u + rad + 1.0) / cs);
  int y0 = (int)floor((v - rad - 1.0) / cs), y1 = (int)floor((v + rad + 1.0) / cs);
  w.x0 = x0 < 0 ? 0 : x0;
  w.y0 = y0 < 0 ? 0 : y0;
  w.x1 = x1 > nx - 1 ? nx - 1 : x1;
  w.y1 = y1 > ny - 1 ? ny - 1 : y1;
  w.u = u;
  w.v = v;
  w.r2 = rad * rad;
  return true;
}

// exact radius / level test + Hamming of one window candidate k; folds (dist, k) into best
__device__ __forceinline__ void gather_test(const lm_fuse_cfg& fc, const PGeo& g, const TgtView& T, const GWin& w,
                                            int k, unsigned long long& best, int* border = nullptr) {
  const double du = T.u[k] - w.u, dv = T.v[k] - w.v;
  const int dl = (int)T.lev[k] - w.lp;
  if (border && (dl < 0 ? -dl : dl) <= fc.level_window) border[0] += near_tie(du * du + dv * dv, w.r2, w.r2);
  if (du * du + dv * dv <= w.r2 && (dl < 0 ? -dl : dl) <= fc.level_window) {
    const int dist = hamming(T.desc[2 * k], T.desc[2 * k + 1], g.r0, g.r1);
    if (dist <= fc.match_max_distance) {
      const unsigned long long key = ((unsigned long long)dist << 32) | (unsigned)k;
      best = key < best ? key : best;
    }
  }
}

// project + gates + grid window search for one (point, target) pair (fusion.py:97-129,
// 178-196). Returns -2 if the point is not visible in the target, -1 if visible without a
// hit, else the hit keypoint (lowest (distance, index) within the window).
__device__ __forceinline__ int gather_hit(const DevMap& M, const lm_fuse_cfg& fc, const PGeo& g, int ts, const TgtView& T,
                          int* border = nullptr) {
  GWin w;
  if (!gather_window(M, fc, g, ts, T, w, border)) return -2;
  unsigned long long best = ~0ull;
  for (int cy = w.y0; cy <= w.y1; ++cy)
    for (int cx = w.x0; cx <= w.x1; ++cx) {
      const int cell = cy * T.nx + cx;
      for (int it = T.cst[cell]; it < T.cst[cell + 1]; ++it) gather_test(fc, g, T, w, T.items[it], best, border);
    }
  return best == ~0ull ? -1 : (int)(best & 0xffffffffu);
}

// the same, warp-cooperative (every lane passes the same point): lane per window cell, so
// the Hamming popcounts of the candidates run side by side instead of on one lane
__device__ int gather_hit_warp(const DevMap& M, const lm_fuse_cfg& fc, const PGeo& g, int ts, const TgtView& T,
                               int lane) {
  GWin w;
  if (!gather_window(M, fc, g, ts, T, w)) return -2;
  const int wx = w.x1 - w.x0 + 1, nc = wx * (w.y1 - w.y0 + 1);
  unsigned long long best = ~0ull;
  for (int c = lane; c < nc; c += 32) {
    const int cy = w.y0 + c / wx, cx = w.x0 + c % wx;
    const int cell = cy * T.nx + cx;
    for (int it = T.cst[cell]; it < T.cst[cell + 1]; ++it) gather_test(fc, g, T, w, T.items[it], best);
  }
  for (int off = 16; off; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
    best = o < best ? o : best;
  }
  return best == ~0ull ? -1 : (int)(best & 0xffffffffu);
}

// fuse_pass action build (fusion.py:161-174) from the hit j, against the current bindings
__device__ __forceinline__ int build_action(const DevMap& M, int pid, int ts, int j, ActRec* act) {
  if (j < 0) return 0;
  const int owner = M.kbind[M.kp_off[ts] + j];
  if (owner < 0) {
    if (observes(M, pid, ts)) return 0;
    *act = ActRec{ts, pid, j, -1, LM_ACT_ADD};
    return 1;
  }
  if (owner != pid && M.alive[owner]) {
    *act = ActRec{ts, pid, j, owner, LM_ACT_MERGE};
    return 1;
  }
  return 0;
}

// fusion borderline counts of this thread into the step record (warp-aggregated)
__device__ __forceinline__ void add_borderline(const DevMap& M, const int border[2]) {
  if (!__any_sync(0xffffffffu, border[0] | border[1])) return;
  int b0 = border[0], b1 = border[1];
  for (int o = 16; o; o >>= 1) {
    b0 += __shfl_xor_sync(0xffffffffu, b0, o);
    b1 += __shfl_xor_sync(0xffffffffu, b1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (b0) atomicAdd((unsigned long long*)&M.s.stats->borderline[2], (unsigned long long)b0);
    if (b1) atomicAdd((unsigned long long*)&M.s.stats->borderline[3], (unsigned long long)b1);
  }
}

__device__ __forceinline__ int gather_one(const DevMap& M, const lm_fuse_cfg& fc, const PGeo& g, int pid, int ts,
                                          const TgtView& T, ActRec* act, int* has_act, int* border = nullptr) {
  const int j = gather_hit(M, fc, g, ts, T, border);
  *has_act = build_action(M, pid, ts, j, act);
  return j >= -1;
}

// ------------------------------------------------------------------ ordered apply
// apply_fusion (fusion.py:249-292) with sequential semantics, executed in parallel by
// deterministic reservations: every round, each pending action reserves every entity it
// would read or write given the current state (its projected point, the hit slot, the
// slot's current owner or the MERGE partner, and when a merge proceeds every slot of the
// loser) with atomicMin of a round-tagged action index; actions holding all their keys
// commit together (their entity sets are disjoint, and no earlier pending action touches
// them), the rest retry. Covisibility bumps are atomic adds and commute.
//
// Points have two access modes. Merges (and ADDs that turn into merges) need a point
// exclusively; a plain ADD only appends a not-yet-observed keyframe to the point, and
// such appends commute with each other (the resulting observation set, counters and
// covisibility deltas do not depend on their order), so ADDs share the point and are
// serialised only against earlier exclusive users. Two ADDs of the same point into the
// same keyframe do not commute (the second is stale); they collide on a hashed
// (point, keyframe) key. Shared-ready ADDs of one point are linked as one group.

enum KeyMode { KM_SLOT = 0, KM_EX = 1, KM_SH = 2, KM_PAIR = 3 };

__device__ __forceinline__ unsigned long long res_tag(unsigned round, int a) {
  return ((unsigned long long)(0xffffffffu - round) << 32) | (unsigned)a;
}

__device__ __forceinline__ int pair_key(int pid, int slot) {
  unsigned h = (unsigned)pid * 0x9E3779B1u + (unsigned)slot * 0x85EBCA77u;
  h ^= h >> 15;
  return (int)(h & (RES_PAIR - 1));
}

// visit the key set of action x under the current state; op(mode, id) -> bool (false stops).
// A key is always visited before the state it guards is read.
template <class Op>
__device__ bool for_keys(const DevMap& M, const ActRec& x, Op op) {
  if (!op(KM_SH, x.pid)) return false;
  if (!M.alive[x.pid] || M.kf_state[x.slot] != KF_LIVE) return true;  // stale
  const int g = M.kp_off[x.slot] + x.j;
  if (!op(KM_SLOT, g)) return false;
  const int now = M.kbind[g];
  int partner = -1;
  if (x.kind == LM_ACT_MERGE) {
    if (!op(KM_EX, x.pid)) return false;
    if (x.other >= 0 && !op(KM_EX, x.other)) return false;
    if (now >= 0 && now != x.other && now != x.pid && !op(KM_EX, now)) return false;
    if (x.other >= 0 && M.alive[x.other] && x.other != x.pid && now == x.other) partner = x.other;
  } else if (now >= 0) {
    if (now != x.pid) {  // the slot was claimed: merge with its owner (or stale)
      if (!op(KM_EX, x.pid) || !op(KM_EX, now)) return false;
      if (M.alive[now]) partner = now;
    }
  } else if (!op(KM_PAIR, pair_key(x.pid, x.slot))) {
    return false;
  }
  if (partner >= 0) {
    const int na = M.nobs[x.pid], nb = M.nobs[partner], fa = M.ooff[x.pid], fb = M.ooff[partner];
    const bool la = na == nb ? x.pid > partner : na < nb;  // the loser's list is the one rebound
    const int2* o = M.obs + (la ? fa : fb);
    const int n = la ? na : nb;
    for (int k0 = 0; k0 < n; k0 += 16) {  // entries and keypoint offsets loaded 16 at a time
      int2 e[16];
      int g[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) e[j] = k0 + j < n ? o[k0 + j] : make_int2(0, 0);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] = k0 + j < n ? M.kp_off[e[j].x] + e[j].y : 0;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j < n && !op(KM_SLOT, g[j])) return false;
    }
  }
  return true;
}

__device__ __forceinline__ void reserve_key(const DevMap& M, int mode, int id, unsigned long long tag) {
  if (mode == KM_SLOT) {
    atomicMin(&M.res_slot[id], tag);
  } else if (mode == KM_PAIR) {
    atomicMin(&M.res_pair[id], tag);
  } else {
    atomicMin(&M.res_pt[id], tag);
    if (mode == KM_EX) atomicMin(&M.res_ex[id], tag);
  }
}

__device__ __forceinline__ bool holds_key(const DevMap& M, int mode, int id, unsigned long long tag) {
  if (mode == KM_SLOT) return M.res_slot[id] == tag;
  if (mode == KM_PAIR) return M.res_pair[id] == tag;
  if (mode == KM_EX) return M.res_pt[id] == tag;
  return M.res_ex[id] >= tag;  // shared: no earlier exclusive user pending
}

// outcome of action x under the current state: 0 stale, 1 add, 2 merge with *partner
__device__ __forceinline__ int classify(const DevMap& M, const ActRec& x, int* partner) {
  if (x.pid < 0 || !M.alive[x.pid] || M.kf_state[x.slot] != KF_LIVE) return 0;
  const int g = M.kp_off[x.slot] + x.j;
  if (x.kind == LM_ACT_MERGE) {
    if (x.other < 0 || !M.alive[x.other] || x.other == x.pid || M.kbind[g] != x.other) return 0;
    *partner = x.other;
    return 2;
  }
  const int now = M.kbind[g];
  if (now >= 0) {
    if (!M.alive[now] || now == x.pid) return 0;
    *partner = now;
    return 2;
  }
  return observes(M, x.pid, x.slot) ? 0 : 1;
}


// A team executes apply_team: one CTA (BlockTeam) or a thread-block cluster (ClusterTeam,
// control words in the leader CTA's shared memory, reached through distributed shared
// memory; barrier.cluster orders global and shared::cluster accesses at cluster scope).
// two banks of control words (round parity): the leader prepares round r + 1's bank while
// round r's later phases read their own, so a round needs no barriers of its own
enum TeamCtl { CTL_ROUND = 0, CTL_NPEND, CTL_NMERGE, CTL_NADD, CTL_NDEF, CTL_NREADY, CTL_NGRPM, CTL_W = 8,
               CTL_N = 2 * CTL_W };

template <int BLOCK>
struct BlockTeam {
  static constexpr int kBlock = BLOCK;
  static constexpr bool kCluster = false;
  int* ctl;
  int tid, nth;
  __device__ explicit BlockTeam(int* c) : ctl(c), tid(threadIdx.x), nth(BLOCK) {}
  __device__ void sync() const { __syncthreads(); }
};

template <int BLOCK>
struct ClusterTeam {
  static constexpr int kBlock = BLOCK;
  static constexpr bool kCluster = true;
  int* ctl;
  int tid, nth, rank, nranks;
  __device__ ClusterTeam(int* local_ctl) {
    cg::cluster_group cl = cg::this_cluster();
    rank = (int)cl.block_rank();
    nranks = (int)cl.num_blocks();
    ctl = cl.map_shared_rank(local_ctl, 0);
    tid = rank * BLOCK + threadIdx.x;
    nth = nranks * BLOCK;
  }
  __device__ void sync() const { cg::this_cluster().sync(); }
};

template <class Team, bool P = true>
__device__ int apply_team(const Team& G, const DevMap& M, const ActRec* acts, int n, int* cnt, int* sh, PairAcc* acc,
                          long long* tm = nullptr) {
  int* const ctl = G.ctl;  // team control words (CTL_*), in the team leader's shared memory
  const int tid = G.tid, nth = G.nth;
  const int lane = threadIdx.x & 31, gwarp = tid >> 5, nwarps = nth >> 5;
  // pend[a]: action a still pending. Done actions are skipped in place (every round walks all
  // n actions: one iteration per thread at these sizes) instead of compacting the pending
  // list with a team-wide scan each round.
  for (int a = tid; a < n; a += nth) M.s.pend[a] = 1;
  // bank `rounds & 1` serves round `rounds`; the leader fills the next round's bank after the
  // check barrier (its words were last read in the round before, ahead of this round's first
  // barrier)
  auto open_bank = [&](int* w, int npend) {
    w[CTL_ROUND] = atomicAdd(&M.scal[SC_ROUND], 1) + 1;
    w[CTL_NPEND] = npend;
    w[CTL_NMERGE] = 0;
    w[CTL_NADD] = 0;
    w[CTL_NDEF] = 0;
    w[CTL_NREADY] = 0;
    w[CTL_NGRPM] = 0;
  };
  if (tid == 0) open_bank(ctl, n);
  G.sync();
  int rounds = 0;
  while (ctl[(rounds & 1) * CTL_W + CTL_NPEND] > 0) {
    int* const cw = ctl + (rounds & 1) * CTL_W;        // this round's words
    int* const nw = ctl + ((rounds + 1) & 1) * CTL_W;  // the next round's
    const int np = cw[CTL_NPEND];
#ifdef LM_DIAG
    if (Team::kCluster && tid == 0) g_diag[17 + (rounds < 4 ? rounds : 4)] += np;
#endif
    if (tm && tid == 0 && rounds > 0) tm[13] += np;  // diagnostics: actions left after round 1
    const unsigned rnd = (unsigned)cw[CTL_ROUND];
    long long tt = gtime_p<P>();
    DIAG_T0
    for (int a = tid; a < n; a += nth) {
      if (!M.s.pend[a]) continue;
      const unsigned long long tag = res_tag(rnd, a);
      const ActRec x = acts[a];
      for_keys(M, x, [&](int mode, int id) {
        reserve_key(M, mode, id, tag);
        return true;
      });
      // every ADD of this round opens its point's ticket counter (same value for all writers);
      // the check phase takes tickets with a plain atomicAdd after the barrier
      if (x.kind == LM_ACT_ADD) M.grp_head[x.pid] = (unsigned long long)rnd << 32;
    }
    DIAG_MAX(0)
    G.sync();
    DIAG_RESTART
    // check (read-only): stale actions are counted, merges queued for warps, ADDs take a
    // ticket in their point's group (gtick = round << 32 | members)
    ActRec my_x{0, 0, 0, 0, 0};
    int my_tick = -1;
    for (int a = tid; a < n; a += nth) {
      if (!M.s.pend[a]) continue;
      const unsigned long long tag = res_tag(rnd, a);
      const ActRec x = acts[a];
      // every key is checked (no early exit): the reservation words load together instead of
      // one dependent load per key (a merge holds a key per observation of its loser)
      bool ready = true;
#ifdef LM_DIAG
      int blocked = -1;
      for_keys(M, x, [&](int mode, int id) {
        const bool h = holds_key(M, mode, id, tag);
        if (!h && blocked < 0) blocked = mode;
        ready &= h;
        return true;
      });
      if (Team::kCluster && blocked >= 0) atomicAdd(&g_diag[24 + blocked + 4 * (x.kind == LM_ACT_MERGE)], 1ull);
#else
      for_keys(M, x, [&](int mode, int id) {
        ready &= holds_key(M, mode, id, tag);
        return true;
      });
#endif
      if (!ready) continue;
      int partner = -1;
      const int kind = classify(M, x, &partner);
      M.s.pend[a] = 0;  // (read by this thread only in this round's loops)
      agg_inc(&cw[CTL_NREADY]);
      if (kind == 0) {
        atomicAdd(&cnt[2], 1);
      } else if (kind == 1) {
        const int tick = (int)(atomicAdd(&M.grp_head[x.pid], 1ull) & 0xffffffffull);
        if (a == tid) {  // the thread's first action stays in registers for the commit phases
          my_x = x;
          my_tick = tick;
        } else {
          const int d = agg_inc(&cw[CTL_NDEF]);
          M.s.def[d] = a;
          M.s.dnxt[d] = tick;
        }
      } else {
        const int at = agg_inc(&cw[CTL_NMERGE]);
        M.s.merge_a[at] = x.pid;
        M.s.merge_b[at] = partner;
        const int na = M.nobs[x.pid], nb = M.nobs[partner];  // (merge_pair_warp's loser rule)
        M.s.die[(na == nb ? x.pid > partner : na < nb) ? x.pid : partner] = (int)rnd;
      }
    }
    DIAG_MAX(1)
    G.sync();
    DIAG_RESTART
#ifdef LM_DIAG
    if (Team::kCluster && tid == 0 && rounds > 0) diag_fold((rounds + 1) & 1);  // the previous round's maxima are final
#endif
    if (tm && tid == 0) {
      tm[9] += gtime_p<P>() - tt;
      tt = gtime_p<P>();
    }
    // group leaders (ticket 0): a lone low-degree ADD links here (thread), a lone high-degree
    // one goes to a warp; a group of m reserves m entries (base = old length) for its members
    const int nd = cw[CTL_NDEF];
    auto head = [&](const ActRec& x, int a_idx) {
      const int p = x.pid;
      const int m = (int)(M.grp_head[p] & 0xffffffffull), n0 = M.nobs[p];
      if (m == 1) {
        if (n0 <= 24) {
          link(M, p, x.slot, x.j, acc, true);
          atomicAdd(&cnt[1], 1);
        } else {
          M.s.add_list[atomicAdd(&cw[CTL_NADD], 1)] = a_idx;
        }
        return;
      }
      if (n0 + m > M.ocap[p]) {  // grow by doubling, copy the current entries
        int nc = M.ocap[p] < 4 ? 4 : M.ocap[p];
        while (nc < n0 + m) nc *= 2;
        const int off = atomicAdd(&M.scal[SC_OBS_HEAD], nc);
        if (off + nc > M.obs_cap) {
          set_err(M, LM_ERR_CAPACITY);
          M.s.gbase[p] = -1;
          return;
        }
        const int2* src = M.obs + M.ooff[p];
        copy_obs(M.obs + off, src, n0);
        M.ooff[p] = off;
        M.ocap[p] = nc;
      }
      M.s.gbase[p] = n0;
      atomicAdd(&cw[CTL_NGRPM], m);
      M.nobs[p] = n0 + m;
      M.found[p] += m;
      M.ver[p] += 1;
      M.gval[p] = 0;
      mark_dirty(M, p);
      atomicAdd(&cnt[1], m);
    };
    if (my_tick == 0) head(my_x, tid);
    for (int d = tid; d < nd; d += nth)
      if (M.s.dnxt[d] == 0ull) head(acts[M.s.def[d]], M.s.def[d]);
    // a pending action whose point (or merge partner) loses a merge of this round is stale:
    // that merge comes first (it holds the point exclusively), and nothing revives a point
    for (int a = tid; a < n; a += nth) {
      if (!M.s.pend[a]) continue;
      const ActRec x = acts[a];
      if ((x.pid >= 0 && M.s.die[x.pid] == (int)rnd) || (x.kind == LM_ACT_MERGE && x.other >= 0 && M.s.die[x.other] == (int)rnd)) {
        M.s.pend[a] = 0;
        agg_inc(&cw[CTL_NREADY]);
        atomicAdd(&cnt[2], 1);
      }
    }
    DIAG_MAX(2)
    G.sync();
    DIAG_RESTART
    if (tid == nth - 1) open_bank(nw, np - cw[CTL_NREADY]);  // (the team's last thread: rarely an action)
    if (tm && tid == 0) {
      tm[10] += gtime_p<P>() - tt;
      tt = gtime_p<P>();
    }
    // group members: own entry, binding, counter, covisibility with the old observers;
    // warps: lone high-degree ADDs and merges (disjoint entities)
    auto member = [&](const ActRec& x, int tick) {
      const int p = x.pid;
      const int m = (int)(M.grp_head[p] & 0xffffffffull);
      const int base = M.s.gbase[p];
      if (m == 1 || base < 0) return;
      int2* o = M.obs + M.ooff[p];
      o[base + tick] = make_int2(x.slot, x.j);
      const int g = M.kp_off[x.slot] + x.j;
      M.kbind[g] = p;
      atomicAdd(&M.counts[(size_t)p * M.L + M.klev[g]], 1);
      covis_list(M, x.slot, o, base, +1, acc);
    };
    if (my_tick >= 0) member(my_x, my_tick);
    for (int d = tid; d < nd; d += nth) member(acts[M.s.def[d]], (int)M.s.dnxt[d]);
    {
      const int nm = cw[CTL_NMERGE], na = cw[CTL_NADD];
      for (int k = gwarp; k < na; k += nwarps) {
        const ActRec x = acts[M.s.add_list[k]];
        link_warp(M, x.pid, x.slot, x.j, lane, acc);  // (found + 1, dirty)
      }
      for (int k = gwarp; k < nm; k += nwarps) merge_pair_warp(M, M.s.merge_a[k], M.s.merge_b[k], lane, acc);
      if (tid == 0) atomicAdd(&cnt[0], nm);
      if (tid == 32) atomicAdd(&cnt[1], na);
    }
    DIAG_MAX(3)
    G.sync();
    DIAG_RESTART
    // group members: covisibility with the members of lower ticket (each new pair once)
    const bool groups = cw[CTL_NGRPM] > 0;
    auto member_pairs = [&](const ActRec& x, int tick) {
      const int p = x.pid;
      const int m = (int)(M.grp_head[p] & 0xffffffffull);
      const int base = M.s.gbase[p];
      if (m == 1 || base < 0) return;
      const int2* o = M.obs + M.ooff[p];
      covis_list(M, x.slot, o + base, tick, +1, acc);
    };
    if (groups && my_tick > 0) member_pairs(my_x, my_tick);
    for (int d = tid; groups && d < nd; d += nth) member_pairs(acts[M.s.def[d]], (int)M.s.dnxt[d]);
    DIAG_MAX(4)
    if (groups) G.sync();
    if (tm && tid == 0) tm[11] += gtime_p<P>() - tt;

    if (++rounds > (1 << 20)) break;
  }
#ifdef LM_DIAG
  if (Team::kCluster && tid == 0 && rounds > 0) diag_fold((rounds + 1) & 1);
#endif
  return rounds;
}


template <int BLOCK, bool P = true>
__device__ int apply_block(const DevMap& M, const ActRec* acts, int n, int* cnt, int* sh, PairAcc* acc,
                           long long* tm = nullptr) {
  __shared__ int ctl[CTL_N];
  const BlockTeam<BLOCK> G(ctl);
  return apply_team<BlockTeam<BLOCK>, P>(G, M, acts, n, cnt, sh, acc, tm);
}

// warp per point of pts[0..P) that is dirty (sort + representative descriptor) or whose
// geometry cache is stale (rebuild), so the per-thread geometry afterwards is O(1)
template <int BLOCK>
__device__ void refresh_points(const DevMap& M, const int* pts, int P, int* sh) {
  int count = 0;
  for (int b0 = 0; b0 < P; b0 += BLOCK) {
    const int p = b0 + threadIdx.x;
    int mp = -1, f = 0;
    if (p < P) {
      mp = pts[p];
      f = mp >= 0 && M.alive[mp] && (M.dirty[mp] || !M.gval[mp]);
    }
    int tot;
    const int at = block_excl_scan<BLOCK>(f, sh, tot);
    if (f) M.s.merge_a[count + at] = mp;  // scratch list (no apply round is in flight)
    count += tot;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = wid; k < count; k += BLOCK / 32) {
    const int mp = M.s.merge_a[k];
    if (M.dirty[mp]) {
      refresh_rep_warp(M, mp, lane);
      if (lane == 0) M.dirty[mp] = 0;
      __syncwarp();
    }
    if (!M.gval[mp]) geo_full_warp(M, mp, lane);
  }
  __syncthreads();
}

// every dirty point of the map (export path)
template <int BLOCK>
__device__ void refresh_all(const DevMap& M) {
  __syncthreads();
  const int n = M.scal[SC_NEXT_ID];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int w0 = wid * 32; w0 < n; w0 += BLOCK) {
    const int id = w0 + lane;
    unsigned bal = __ballot_sync(0xffffffffu, id < n && M.dirty[id]);
    while (bal) {
      const int k = __ffs(bal) - 1;
      bal &= bal - 1;
      const int mp = w0 + k;
      if (M.alive[mp]) refresh_rep_warp(M, mp, lane);
      __syncwarp();
      if (lane == 0) M.dirty[mp] = 0;
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) M.scal[SC_DIRTY_N] = 0;
  __syncthreads();
}

// bound live points of keyframe slot (mapmodel.py:291-300), in keypoint order, into M.s.pts
template <int BLOCK>
__device__ int bound_points(const DevMap& M, int slot, int* sh) {
  const int off = M.kp_off[slot], n = M.kp_n[slot];
  int count = 0;
  for (int b0 = 0; b0 < n; b0 += BLOCK) {
    const int i = b0 + threadIdx.x;
    int mp = -1, f = 0;
    if (i < n) {
      mp = M.kbind[off + i];
      f = mp >= 0 && M.alive[mp];
    }
    int tot;
    const int at = block_excl_scan<BLOCK>(f, sh, tot);
    if (f) M.s.pts[count + at] = mp;
    count += tot;
  }
  __syncthreads();
  return count;
}

// collect_fusion_targets (fusion.py:38-54): first-order neighbours in rank order, then per
// first-order keyframe (in order) up to n2 not-yet-listed keyframes of its own ranking.
// Every first-order row is ranked in parallel (warp per row, 64-bit composite keys); the
// dependent walk is one thread over shared memory with a slot bitmap for "seen".
template <int BLOCK>
__device__ int fusion_targets(const DevMap& M, int cur, int n1, int n2, int n_slots, int* sh_slot,
                              unsigned long long* sh_key) {
  __shared__ int first[TMAX];
  __shared__ int tlist[TMAX];
  __shared__ int n_first, n_t;
  // per slot: already a target (plain byte stores), in the dynamic area after sh_slot
  unsigned char* seen = (unsigned char*)(sh_slot + M.kf_cap);
  constexpr int HR = 64;          // rows whose 32 best-ranked entries are kept in shared memory
  __shared__ int head[HR][32], hcnt[HR];
  const int nf = ranked_neighbors<BLOCK>(M, cur, n1 < TMAX ? n1 : TMAX, sh_slot, sh_key, first, n_slots);
  if (threadIdx.x == 0) n_first = nf;
  for (int k = threadIdx.x; k < n_slots; k += BLOCK) seen[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t stride = 3 * (size_t)M.kf_cap + 1;
  for (int f = wid; f < n_first; f += BLOCK / 32) {
    // rank_buf row: [count][slot x kf_cap][ranked slot x kf_cap][key (u64) x kf_cap/2...]
    int* buf = M.s.rank_buf + (size_t)f * stride;
    unsigned long long* keys = (unsigned long long*)(M.s.rank_buf + (size_t)TMAX * stride) + (size_t)f * M.kf_cap;
    const int row_slot = first[f];
    const int* row = M.covis + (size_t)row_slot * M.kf_cap;
    int c = 0;
    constexpr int PF = 8;  // row chunks whose loads are issued together (one L2 round trip per 8)
    for (int s00 = 0; s00 < n_slots; s00 += 32 * PF) {
      int wv[PF], st[PF];
      long long kid[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int s = s00 + 32 * u + lane;
        wv[u] = s < n_slots ? __ldcg(row + s) : 0;  // (L2, see ranked_neighbors)
        st[u] = s < n_slots ? M.kf_state[s] : 0;
        kid[u] = s < n_slots ? M.kf_id[s] : 0;
      }
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int s = s00 + 32 * u + lane;
        const int w = wv[u];
        const bool take = s < n_slots && s != row_slot && w >= M.min_w && w > 0 && st[u] == KF_LIVE;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (take) {
          const int at = c + __popc(bal & ((1u << lane) - 1));
          buf[1 + at] = s;
          keys[at] = ((unsigned long long)(0x7fffffff - w) << 32) | (unsigned)kid[u];  // covis_key
        }
        c += __popc(bal);
      }
    }
    __syncwarp();
    for (int e = lane; e < c; e += 32) {
      const unsigned long long ke = keys[e];
      int rk = 0;
      for (int q = 0; q < c; ++q) rk += keys[q] < ke;
      buf[1 + M.kf_cap + rk] = buf[1 + e];
      if (f < HR && rk < 32) head[f][rk] = buf[1 + e];
    }
    if (lane == 0) {
      buf[0] = c;
      if (f < HR) hcnt[f] = c;
    }
    __syncwarp();
  }
  __syncthreads();
  if (wid == 0) {  // the dependent walk, one warp: lanes test 32 ranked candidates at once
    for (int f = lane; f < n_first; f += 32) {
      tlist[f] = first[f];
      seen[first[f]] = 1;
    }
    if (lane == 0) seen[cur] = 1;
    __syncwarp();
    int nt = n_first;
    for (int f = 0; f < n_first; ++f) {
      const int* buf = M.s.rank_buf + (size_t)f * stride;
      const int c = f < HR ? hcnt[f] : buf[0];
      int added = 0;
      for (int q0 = 0; q0 < c && added < n2 && nt < TMAX; q0 += 32) {
        const int q = q0 + lane;
        const int sl = q < c ? (f < HR && q < 32 ? head[f][q] : buf[1 + M.kf_cap + q]) : -1;
        const bool un = sl >= 0 && !seen[sl];
        const unsigned bal = __ballot_sync(0xffffffffu, un);
        const int want = n2 - added < TMAX - nt ? n2 - added : TMAX - nt;
        const int rk = __popc(bal & ((1u << lane) - 1));
        if (un && rk < want) {
          tlist[nt + rk] = sl;
          seen[sl] = 1;
        }
        const int got = __popc(bal) < want ? __popc(bal) : want;
        nt += got;
        added += got;
        __syncwarp();
      }
    }
    if (lane == 0) {
      n_t = nt;
      *M.s.n_targets = nt;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n_t; k += BLOCK) M.s.targets[k] = tlist[k];
  __syncthreads();
  return n_t;
}

// points M.s.pts[0..P) into target ts: refresh, geometry, gather, (visible), compaction
template <int BLOCK>
__device__ int gather_pass(const DevMap& M, const lm_fuse_cfg& fc, int P, int ts, const TgtView& TV,
                           bool bump_visible, int* sh, int* vis_out, long long* tm = nullptr) {
  const long long c0 = gtime();
  refresh_points<BLOCK>(M, M.s.pts, P, sh);
  if (tm && threadIdx.x == 0) tm[0] += gtime() - c0;
  const long long c1 = gtime();
  for (int p = threadIdx.x; p < P; p += BLOCK) point_geometry(M, M.s.pts[p], fc.dist_band_slack, M.s.geo[p]);
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[1] += gtime() - c1;
  const long long c2 = gtime();
  int count = 0, nvis = 0;
  for (int b0 = 0; b0 < P; b0 += BLOCK) {
    const int p = b0 + threadIdx.x;
    ActRec a;
    int has = 0, vis = 0;
    if (p < P) {
      const int pid = M.s.pts[p];
      vis = gather_one(M, fc, M.s.geo[p], pid, ts, TV, &a, &has);
      if (vis && bump_visible && M.alive[pid]) atomicAdd(&M.visible[pid], 1);
      if (vis_out) M.s.vis_flag[p] = vis;
    }
    int tot;
    const int at = block_excl_scan<BLOCK>(has, sh, tot);
    if (has) M.s.acts[count + at] = a;
    count += tot;
    nvis += vis;
  }
  if (vis_out) *vis_out = block_sum<BLOCK>(nvis, sh);
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[3] += gtime() - c2;
  return count;
}


// per pass 56 B per point (pos 24 + rep 32), 9 B per observation, 53 B per
// target keypoint (u,v 16 + level 1 + desc 32 + binding 4), 16 B per action
__device__ __forceinline__ long long pass_bytes(long long pts, long long obs, long long tkp, long long acts) {
  return 56 * pts + 9 * obs + 53 * tkp + 16 * acts;
}

enum FuseCtl { FC_T = 0, FC_P = 1, FC_NACT = 2, FC_NU = 3, FC_NSP = 4, FC_DONE = 5, FC_N = 8 };

// Starts while its predecessor (k_commit_write: the new points' records and the current
// keyframe's new bindings) still runs: target selection reads only covisibility, which
// k_commit wrote before k_commit_write started; the wait comes right before the current
// keyframe's bound points are read (and on every exit path, so completion stays ordered).
__global__ void __launch_bounds__(1024) k_fuse_targets(DevMap* maps, const StepArgs* args, int n_slots_max) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const StepArgs& A = args[blockIdx.x];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  extern __shared__ unsigned long long dynk[];
  unsigned long long* sh_key = dynk;
  int* sh_slot = (int*)(dynk + M.kf_cap);
  __shared__ int sh[32];
  const long long t0 = gtime();
  int T = fusion_targets<1024>(M, A.cur, A.fc.n1, A.fc.n2, n_slots_max, sh_slot, sh_key);
  {  // record_neighbor_access("fusion", targets): all resident, else the stage fails untouched
    int bad = 0;
    const bool enforce = !M.scal[SC_NORES];
    for (int k = threadIdx.x; k < T; k += 1024) bad |= enforce && !M.kf_res[M.s.targets[k]];
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) atomicCAS(&M.scal[SC_SOFT], 0, LM_ERR_INVALID_STATE);
      T = 0;
    }
  }
  __shared__ unsigned long long s_tkp;
  if (threadIdx.x == 0) s_tkp = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_commit_write's bindings from here on
  const int P = T ? bound_points<1024>(M, A.cur, sh) : 0;  // (barriers)
  {  // keypoints of the targets, block-parallel
    int tk = 0;
    for (int k = threadIdx.x; k < T; k += 1024) tk += M.kp_n[M.s.targets[k]];
    for (int off = 16; off; off >>= 1) tk += __shfl_xor_sync(0xffffffffu, tk, off);
    if ((threadIdx.x & 31) == 0 && tk) atomicAdd(&s_tkp, (unsigned long long)tk);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    M.s.fctl[FC_T] = T;
    M.s.fctl[FC_P] = P;
    lm_step_stats* st = M.s.stats;
    st->n_targets = T;
    if (T) {
      const unsigned long long mpb = M.mp_rec_bytes;
      const long long tkp = (long long)s_tkp;
      const unsigned long long ev = M.ledger[LG_SMALL_EVENTS];
      if (ev < (unsigned long long)LG_LOG_CAP) M.lg_log[ev] = (long long)(P * mpb);
      const unsigned long long naive = (unsigned long long)tkp * (M.kp_rec_bytes + M.desc_bytes);  // payload_bytes
      M.ledger[LG_NAIVE] += naive + P * mpb;
      M.ledger[LG_PERSIST] += P * mpb;
      M.ledger[LG_SMALL_FUSE] += P * mpb;
      M.ledger[LG_SMALL_EVENTS] += 1;
      st->fuse_points += (long long)T * P;
      st->fuse_passes += T;
      st->fuse_bytes += 53 * tkp;
    }
    st->fuse_cycles[0] += gtime() - t0;
  }
}

// warp per forward point: refresh a stale rep descriptor, then the geometry row
__global__ void __launch_bounds__(256) k_fuse_geo(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  const int P = M.s.fctl[FC_P];
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (blockIdx.x * 8 >= P) return;  // (whole block: uniform)
  const int mp = p < P ? M.s.pts[p] : -1;
  if (mp >= 0 && M.alive[mp]) {
    if (M.dirty[mp]) {
      refresh_rep_warp(M, mp, lane);
      if (lane == 0) M.dirty[mp] = 0;
      __syncwarp();
    }
    if (!M.gval[mp]) geo_full_warp(M, mp, lane);
  }
  __shared__ unsigned long long fb_sh;
  if (threadIdx.x == 0) fb_sh = 0;
  __syncthreads();
  if (lane == 0 && mp >= 0) {
    point_geometry(M, mp, A.fc.dist_band_slack, M.s.geo[p]);
    atomicAdd(&fb_sh, (unsigned long long)(M.s.fctl[FC_T] * (56LL + 9LL * M.nobs[mp])));
  }
  __syncthreads();  // algorithmic bytes: one same-address global atomic per block, not per point
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)&M.s.stats->fuse_bytes, fb_sh);
}

// thread per (target, point) of the forward gather; per-CTA ordered compaction
__global__ void __launch_bounds__(256) k_fuse_gather(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  __shared__ int sh[32];
  const int T = M.s.fctl[FC_T], P = M.s.fctl[FC_P];
  const int TP = T * P;
  const int b0 = blockIdx.x * 256;
  if (b0 >= TP) return;
  const int it = b0 + threadIdx.x;
  ActRec a;
  int has = 0;
  int border[2] = {0, 0};
  if (it < TP) {
    const int t = it / P, p = it - t * P;
    const int pid = M.s.pts[p];
    const int ts = M.s.targets[t];
    if (gather_one(M, A.fc, M.s.geo[p], pid, ts, tgt_global(M, ts), &a, &has, border)) atomicAdd(&M.visible[pid], 1);
  }
  add_borderline(M, border);
  int tot;
  const int at = block_excl_scan<256>(has, sh, tot);
  if (has) M.s.acts2[b0 + at] = a;
  if (threadIdx.x == 0) M.s.blk_cnt[blockIdx.x] = tot;
}

// assemble the forward batch in (target, point) order and apply it
constexpr int APPLY_THREADS = 512;  // k_fuse_apply CTA (128 registers: apply_team does not spill)

// Forward apply: one thread-block cluster per map (launched with cluster dims; blockIdx.x /
// cluster size selects the map). The ~4.5k forward actions of a C2 keyframe spread over the
// cluster's CTAs; the reservation rounds synchronise with barrier.cluster.
template <bool TP>
__global__ void __launch_bounds__(APPLY_THREADS, 1) k_fuse_apply(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  cg::cluster_group cl = cg::this_cluster();
  const int ncl = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const StepArgs& A = args[blockIdx.x / ncl];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  const int T = M.s.fctl[FC_T], P = M.s.fctl[FC_P];
  if (T == 0) return;
  __shared__ int sh[32];
  __shared__ int cnt[3];
  __shared__ int ctl[CTL_N];
  __shared__ PairAcc acc;
  __shared__ long long tmf[16];
  const long long t0 = gtime_p<TP>();
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  if (threadIdx.x < 16) tmf[threadIdx.x] = 0;
  pair_acc_init<APPLY_THREADS>(&acc, A.cur);
  const ClusterTeam<APPLY_THREADS> G(ctl);
  const int nb = (T * P + 255) / 256;
  int base = 0;
  for (int c0 = 0; c0 < nb; c0 += APPLY_THREADS) {  // exclusive scan of the per-CTA counts (every CTA)
    const int b = c0 + threadIdx.x;
    const int v = b < nb ? M.s.blk_cnt[b] : 0;
    int tot;
    const int at = block_excl_scan<APPLY_THREADS>(v, sh, tot);
    if (b < nb && rank == 0) M.s.blk_off[b] = base + at;
    base += tot;
  }
  const int nact = base;
  G.sync();
  for (int b = G.tid >> 5; b < nb; b += G.nth >> 5) {  // warp per source CTA segment
    const int c = M.s.blk_cnt[b], o = M.s.blk_off[b];
    for (int k = threadIdx.x & 31; k < c; k += 32) M.s.acts[o + k] = M.s.acts2[b * 256 + k];
  }
  G.sync();
  const long long t1 = gtime_p<TP>();
  const int rr = apply_team<ClusterTeam<APPLY_THREADS>, TP>(G, M, M.s.acts, nact, cnt, sh, &acc, rank == 0 ? tmf : nullptr);
  pair_acc_flush<APPLY_THREADS>(M, &acc);
  lm_step_stats* st = M.s.stats;
  if (threadIdx.x == 0) {
    atomicAdd(&st->merged, cnt[0]);
    atomicAdd(&st->observations_added, cnt[1]);
    atomicAdd(&st->stale, cnt[2]);
  }
  if (G.tid == 0) {
    st->fuse_actions += nact;
    st->fuse_bytes += 16LL * nact;
    st->apply_rounds += rr;
    st->fuse_cycles[2] += t1 - t0;
    st->fuse_cycles[3] += gtime_p<TP>() - t1;
    st->fuse_cycles[13] += tmf[9];   // forward: reserve+check
    st->fuse_cycles[14] += tmf[10] + tmf[11];  // forward: commit (plain + merges)
    st->fuse_cycles[15] += tmf[12];  // forward: compaction
    st->dbg[8] += tmf[10];           // forward: group leaders (heads)
    st->dbg[9] += tmf[11];           // forward: members / merges / member pairs
    st->dbg[10] += rr;               // forward: rounds
    st->dbg[11] += nact;             // forward: actions
    st->dbg[15] += tmf[13];          // forward: actions pending in rounds 2..
  }
  cl.sync();  // the leader CTA's shared control words stay alive until every CTA is done
}

// ---------------------------------------------------------------------- reverse passes
// Reference: for t in targets: gather(bound_points_of(t) -> current) then apply
// (fusion.py:337-346) -- each pass sees every earlier pass's mutations. Only a few passes
// produce actions (C2: ~6 of ~75), and a pass without actions changes nothing but visible
// counters, so passes are evaluated speculatively, item by item ((pass, keypoint)):
//   k_fuse_spec    evaluates every item against the post-forward map (thread per item):
//                  the bound point, its hit into the current keyframe, its action, and per
//                  current keypoint j the bitmap of passes hitting j.
//   k_fuse_rev     (one CTA per map) walks to the first pass with actions, applies it, and
//                  re-evaluates exactly the later items whose inputs that apply touched,
//                  updating the per-pass totals by deltas; repeats until no pass acts.
//   k_fuse_visible commits every pass's visible counters (thread per item).
// An item's inputs are the binding of its keypoint, that point's state (version), and the
// binding of the current keypoint it hits. An apply changes the state of the points of its
// actions and of their slot owners (the "touched" points); the bindings that change are
// the touched points' slots before or after the apply (touched items) and current
// keypoints (found by comparing with a snapshot; items hitting them are found through the
// pass bitmap). Visible bumps are deferred: a bump of a point that a later merge kills is
// the same as a bump of its winner after the merge (the merge sums the counters), so
// k_fuse_visible follows the loser -> winner records of this step (mrg, SC_MTAG).

constexpr int HPW = (TMAX + 31) / 32;  // words of the per-current-keypoint pass bitmap
constexpr int REV_THREADS = 512;       // k_fuse_rev block (128 registers: the register-resident refresh must not spill)
enum PassInfo { PI_NACT = 0, PI_LIVE = 1, PI_OBS = 2, PI_N = 3 };

// warp per point touched since the last refresh: representative descriptor + geometry cache;
// also clears the reverse-pass bookkeeping for k_fuse_spec
__global__ void __launch_bounds__(256) k_fuse_refresh(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  {
    const int tid = blockIdx.x * 256 + threadIdx.x, nth = gridDim.x * 256;
    for (int k = tid; k < PI_N * TMAX; k += nth) M.s.pinfo[k] = 0;
    for (int k = tid; k < M.kpkf_max * HPW; k += nth) M.s.hitpass[k] = 0u;
    for (int k = tid; k < M.kpkf_max; k += nth) M.s.hl_cnt[k] = 0;
    const int aw_all = M.s.fctl[FC_T] * ((M.kpkf_max + 31) >> 5);
    for (int k = tid; k < aw_all; k += nth) M.s.abits[k] = 0u;
    if (tid == 0) {
      M.scal[SC_MTAG] += 1;  // merges of this step's reverse phase
      M.s.fctl[FC_NU] = 0;
      M.s.fctl[FC_NSP] = 0;
    }
  }
  const int n = M.scal[SC_DIRTY_N];
  const int lane = threadIdx.x & 31;
  for (int k = blockIdx.x * 8 + (threadIdx.x >> 5); k < n; k += gridDim.x * 8) {
    const int mp = M.dirty_list[k];
    // the list can hold a point twice (dirty again after an earlier refresh): one warp
    // claims it, so no two warps sort the same observation list
    int claim = 0;
    if (lane == 0) claim = atomicExch(&M.dirty[mp], 0);
    if (!__shfl_sync(0xffffffffu, claim, 0)) continue;
    if (M.alive[mp]) {
      refresh_rep_warp(M, mp, lane);
      if (!M.gval[mp]) geo_full_warp(M, mp, lane);
    }
  }
}

// register point mp under its hit j in the per-keypoint hit list
__device__ __forceinline__ void hit_list_add(const DevMap& M, int j, int mp) {
  if (j < 0) return;
  const int at = atomicAdd(&M.s.hl_cnt[j], 1);
  if (at < HL) M.s.hl[j * HL + at] = mp;
}

struct ItemVal {
  int mp, j, nob, has;
  ActRec a;
};

// evaluate item (pass t, keypoint kp of target ts) on the current state; the bound point's
// cached hit must be current. Records the hit bit of the pass.
__device__ __forceinline__ ItemVal eval_item(const DevMap& M, int cur, int t, int ts, int kp) {
  ItemVal v{-1, -3, 0, 0, ActRec{0, 0, 0, 0, 0}};
  const int mp = M.kbind[M.kp_off[ts] + kp];
  if (mp >= 0 && M.alive[mp]) {
    v.mp = mp;
    v.nob = M.nobs[mp];
    v.j = M.hit[mp].y;
    if (v.j >= 0) {
      atomicOr(&M.s.hitpass[v.j * HPW + (t >> 5)], 1u << (t & 31));
      v.has = build_action(M, mp, cur, v.j, &v.a);
    }
  }
  return v;
}

__device__ __forceinline__ void store_item(const DevMap& M, size_t it, const ItemVal& v) {
  M.s.pj[it] = v.j;
  M.s.pmp[it] = v.mp;
  M.s.pob[it] = v.nob;
  ActRec a = v.a;
  if (!v.has) a.kind = 0;
  M.s.acts2[it] = a;
}

// speculative evaluation of every reverse-pass item on the post-forward map, in three wide
// kernels: the distinct bound points of all passes (a point is bound in up to ~all targets,
// and its hit into the current keyframe does not depend on the pass), their hits, the items

// (1) thread per (pass, keypoint): each live bound point joins the distinct list once
__global__ void __launch_bounds__(256) k_fuse_spec_pts(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  const int t = blockIdx.y;
  if (t >= M.s.fctl[FC_T]) return;
  const int ts = M.s.targets[t];
  const int kp = blockIdx.x * 256 + threadIdx.x;
  if (kp >= M.kp_n[ts]) return;
  const int mp = M.kbind[M.kp_off[ts] + kp];
  if (mp < 0 || !M.alive[mp]) return;
  const int stag = M.scal[SC_MTAG];
  if (atomicExch(&M.s.hreg[mp], stag) != stag) M.s.upts[atomicAdd(&M.s.fctl[FC_NU], 1)] = mp;
}

// (2) thread per distinct point (grid-stride): geometry, window search, hit list
__global__ void __launch_bounds__(256) k_fuse_spec_hit(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  if (M.s.fctl[FC_T] == 0) return;
  const int nu = M.s.fctl[FC_NU];
  const TgtView T = tgt_global(M, A.cur);
  for (int k = blockIdx.x * 256 + threadIdx.x; k < nu; k += gridDim.x * 256) {
    const int mp = M.s.upts[k];
    PGeo g;
    point_geometry(M, mp, A.fc.dist_band_slack, g);
    int border[2] = {0, 0};
    const int j = gather_hit(M, A.fc, g, A.cur, T, border);
    M.hit[mp] = make_int2(M.ver[mp], j);
    hit_list_add(M, j, mp);
    if (border[0]) atomicAdd((unsigned long long*)&M.s.stats->borderline[2], (unsigned long long)border[0]);
    if (border[1]) atomicAdd((unsigned long long*)&M.s.stats->borderline[3], (unsigned long long)border[1]);
  }
}

// (3) thread per (pass, keypoint): the item (bound point, hit, action), pass totals. With
// GATHER (a single session: launches cost more than the redundant gathers) the item computes
// its point's hit itself and (1)/(2) are skipped.
template <bool GATHER>
__global__ void __launch_bounds__(256) k_fuse_spec(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.z];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;
  const int t = blockIdx.y;
  if (t >= M.s.fctl[FC_T]) return;
  const int ts = M.s.targets[t];
  const int n = M.kp_n[ts];
  if ((int)blockIdx.x * 256 >= n) return;
  const int kp = blockIdx.x * 256 + threadIdx.x;
  int live = 0, nob = 0, has = 0;
  if (kp < n) {
    if (GATHER) {
      const int mp = M.kbind[M.kp_off[ts] + kp];
      if (mp >= 0 && M.alive[mp]) {  // identical values from every pass binding the point
        PGeo g;
        point_geometry(M, mp, A.fc.dist_band_slack, g);  // caches valid (k_fuse_refresh)
        int border[2] = {0, 0};
        const int j = gather_hit(M, A.fc, g, A.cur, tgt_global(M, A.cur), border);
        M.hit[mp] = make_int2(M.ver[mp], j);
        const int stag = M.scal[SC_MTAG];
        // every pass binding the point computes the same (j, border); the first one to
        // register it lists the hit and counts its borderline compares
        if ((j >= 0 || (border[0] | border[1])) && atomicExch(&M.s.hreg[mp], stag) != stag) {
          if (j >= 0) hit_list_add(M, j, mp);
          if (border[0]) atomicAdd((unsigned long long*)&M.s.stats->borderline[2], (unsigned long long)border[0]);
          if (border[1]) atomicAdd((unsigned long long*)&M.s.stats->borderline[3], (unsigned long long)border[1]);
        }
      }
    }
    const ItemVal v = eval_item(M, A.cur, t, ts, kp);
    store_item(M, (size_t)t * M.kpkf_max + kp, v);
    if (v.has) atomicOr(&M.s.abits[(size_t)t * ((M.kpkf_max + 31) >> 5) + (kp >> 5)], 1u << (kp & 31));
    if (v.has && v.a.kind == LM_ACT_ADD) {  // post-ADD state of this point, precomputed by k_fuse_post
      const int stag = M.scal[SC_MTAG];
      if (atomicExch(&M.sp_tag[v.mp], stag) != stag) {
        M.sp_j[v.mp] = v.a.j;
        M.s.sp_list[atomicAdd(&M.s.fctl[FC_NSP], 1)] = v.mp;
      }
    }
    live = v.mp >= 0;
    nob = v.nob;
    has = v.has;
  }
  for (int off = 16; off; off >>= 1) {
    live += __shfl_xor_sync(0xffffffffu, live, off);
    nob += __shfl_xor_sync(0xffffffffu, nob, off);
    has += __shfl_xor_sync(0xffffffffu, has, off);
  }
  if ((threadIdx.x & 31) == 0 && live) {
    atomicAdd(&M.s.pinfo[PI_LIVE * TMAX + t], live);
    atomicAdd(&M.s.pinfo[PI_OBS * TMAX + t], nob);
    if (has) atomicAdd(&M.s.pinfo[PI_NACT * TMAX + t], has);
  }
}

// Speculative post-ADD states. Most reverse-pass actions are ADDs of a point into the
// current keyframe, and each such point's state after that ADD (observations + (cur, j))
// is known before the reverse walk starts: its representative descriptor, view geometry
// and new hit are computed here, wide (warp per point). k_fuse_rev takes them instead of
// refreshing when the apply did exactly that (one mutation, one observation more, slot j
// bound to the point: the same observation set).
constexpr int POST_MAXN = 128;
constexpr int POST_BLOCKS = 148;  // k_fuse_post grid (x) upper bound: scratch per warp (LM_POST_BLOCKS; 296 measured no faster)
__global__ void __launch_bounds__(256) k_fuse_post(DevMap* maps, const StepArgs* args) {
  pdl_enter();
  const StepArgs& A = args[blockIdx.y];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse || M.s.fctl[FC_T] == 0) return;
  const int nsp = M.s.fctl[FC_NSP];
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5), nw = gridDim.x * 8;
  int2* scratch = M.s.sp_obs + (size_t)gw * (POST_MAXN + 1);
  const int cur = A.cur;
  const TgtView T = tgt_global(M, cur);
  for (int k = gw; k < nsp; k += nw) {
    const int p = M.s.sp_list[k];
    const int n0 = M.nobs[p], j = M.sp_j[p];
    if (!M.alive[p] || n0 + 1 > POST_MAXN) {
      if (lane == 0) M.sp_ver0[p] = -1;
      continue;
    }
    if (!M.gval[p]) geo_full_warp(M, p, lane);  // (current-state cache: a pure function)
    const int2* o = M.obs + M.ooff[p];
    for (int e = lane; e < n0; e += 32) scratch[e] = o[e];
    if (lane == 0) scratch[n0] = make_int2(cur, j);
    __syncwarp();
    refresh_rep_list(M, scratch, n0 + 1, M.sp_rep + 2 * (size_t)p, lane);
    __syncwarp();
    // geometry: the current keyframe is the newest, so its term extends the sums exactly
    double ax = M.gacc[3 * p], ay = M.gacc[3 * p + 1], az = M.gacc[3 * p + 2], lo = M.glo[p], hi = M.ghi[p];
    const double rx = M.pos[3 * p] - M.C[3 * cur], ry = M.pos[3 * p + 1] - M.C[3 * cur + 1];
    const double rz = M.pos[3 * p + 2] - M.C[3 * cur + 2];
    const double dd = sqrt(rx * rx + ry * ry + rz * rz);
    if (dd > 0) {
      const double d0 = dd / M.S[M.klev[M.kp_off[cur] + j]];
      lo = d0 < lo ? d0 : lo;
      hi = d0 > hi ? d0 : hi;
      ax = ax + rx / dd;
      ay = ay + ry / dd;
      az = az + rz / dd;
    }
    PGeo g;
    g.ok = 0;
    if (isfinite(lo)) {
      const double nrm = sqrt(ax * ax + ay * ay + az * az);
      g.vx = nrm > 0 ? ax / nrm : ax;
      g.vy = nrm > 0 ? ay / nrm : ay;
      g.vz = nrm > 0 ? az / nrm : az;
      g.x = M.pos[3 * p];
      g.y = M.pos[3 * p + 1];
      g.z = M.pos[3 * p + 2];
      g.d0 = lo;
      g.blo = lo / A.fc.dist_band_slack;
      g.bhi = hi * M.S[M.L - 1] * A.fc.dist_band_slack;
      g.r0 = M.sp_rep[2 * (size_t)p];
      g.r1 = M.sp_rep[2 * (size_t)p + 1];
      g.ok = 1;
    }
    const int hit = gather_hit_warp(M, A.fc, g, cur, T, lane);
    if (lane == 0) {
      double* sg = M.sp_geo + 5 * (size_t)p;
      sg[0] = ax;
      sg[1] = ay;
      sg[2] = az;
      sg[3] = lo;
      sg[4] = hi;
      M.sp_hit[p] = hit;
      M.sp_ver0[p] = M.ver[p];
      M.sp_nobs0[p] = n0;
    }
    __syncwarp();
  }
}

// reverse passes (fusion.py:337-346), one CTA per map; see the block comment above
template <bool P>
__global__ void __launch_bounds__(REV_THREADS, 1) k_fuse_rev(DevMap* maps, const StepArgs* args, int smem_bytes, int wide) {
  pdl_enter();
  // one cluster per map: CTA 0 walks the passes; the other CTAs (if any) only help apply the
  // direct passes' actions, on command (rcmd in CTA 0's shared memory, cluster barriers)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), nranks = (int)cl.num_blocks();
  const StepArgs& A = args[blockIdx.x / nranks];
  const DevMap& M = maps[A.map];
  if (!A.do_fuse) return;  // (uniform over the cluster)
  const int T = M.s.fctl[FC_T];
  if (T == 0) return;
  const long long t_entry = gtime_p<P>();
  extern __shared__ __align__(16) unsigned char dyn_rev[];
  TgtView TV = tgt_global(M, A.cur);
  {  // stage the current keyframe (target of every reverse pass) in shared memory
    const int n = M.kp_n[A.cur], off = M.kp_off[A.cur];
    const int nc = M.g_nx[A.cur] * M.g_ny[A.cur];
    const size_t need = (size_t)n * 53 + 4 * (size_t)(nc + 1) + 64;
    if (rank == 0 && smem_bytes > 0 && need <= (size_t)smem_bytes) {
      uint4* sd = (uint4*)dyn_rev;
      double* su = (double*)(sd + 2 * n);
      double* sv = su + n;
      int* scs = (int*)(sv + n);
      int* sit = scs + nc + 1;
      unsigned char* sl = (unsigned char*)(sit + n);
      for (int k = threadIdx.x; k < 2 * n; k += REV_THREADS) sd[k] = M.kdesc[2 * (size_t)off + k];
      for (int k = threadIdx.x; k < n; k += REV_THREADS) {
        su[k] = M.ku[off + k];
        sv[k] = M.kv[off + k];
        sit[k] = M.cell_items[off + k];
        sl[k] = M.klev[off + k];
      }
      const int* gcs = M.cell_start + (size_t)A.cur * (GRID_CELLS + 1);
      for (int k = threadIdx.x; k <= nc; k += REV_THREADS) scs[k] = gcs[k];
      TV = TgtView{su, sv, sl, sd, scs, sit, nullptr, TV.nx, TV.ny};
    }
  }
  __shared__ int sh[32];
  __shared__ int cnt[3];
  __shared__ long long tm[16];
  __shared__ PairAcc acc;
  __shared__ int s_nact[TMAX], s_live[TMAX], s_obs[TMAX];
  __shared__ int t1_sh, nc_sh, ni_sh, tag_sh, tmin_sh, na_sh, nchg_sh, fast_sh;
  constexpr int DMAX = 128;  // largest direct pass
  constexpr int JBW = 64;    // words of the direct pass's keypoint bitmap
  __shared__ int s_inst[DMAX];  // direct pass: action k's point took its speculated state
  __shared__ unsigned s_jb[JBW];
  __shared__ int s_nset, tag_base;
  constexpr int ILS = 1024;
  __shared__ int s_il[ILS];     // the iteration's item list (overflow: M.s.ilist)
  __shared__ int s_toff[TMAX];  // keypoint offset of each pass's target
  __shared__ ActRec s_acts[DMAX];  // the pass's first DMAX actions
  __shared__ double cur_pose[22];  // R, t, C, cam, cell size of the current keyframe
  __shared__ int rcmd[5];          // CTA 0 -> helpers: command, t1, tag, action / point count, ncand
  enum { RC_DIRECT = 1, RC_EXIT = 2, RC_SETTLE = 3, RC_RESCAN = 4, RC_PTITEMS = 5, RC_HITLIST = 6 };
  // CTA 0's counters and lists, reached by the helper CTAs through distributed shared memory
  int* const ni_p = rank ? cl.map_shared_rank(&ni_sh, 0) : &ni_sh;
  int* const nset_p = rank ? cl.map_shared_rank(&s_nset, 0) : &s_nset;
  int* const il_p = rank ? cl.map_shared_rank(s_il, 0) : s_il;
  int* const inst_p = rank ? cl.map_shared_rank(s_inst, 0) : s_inst;
  const int* const rcmd0 = cl.map_shared_rank(rcmd, 0);
  int* const live_p = rank ? cl.map_shared_rank(s_live, 0) : s_live;
  int* const obs_p = rank ? cl.map_shared_rank(s_obs, 0) : s_obs;
  int* const nact_p = rank ? cl.map_shared_rank(s_nact, 0) : s_nact;
  int* const tmin_p = rank ? cl.map_shared_rank(&tmin_sh, 0) : &tmin_sh;
  int* const nc_p = rank ? cl.map_shared_rank(&nc_sh, 0) : &nc_sh;
  if (threadIdx.x < 22) {
    const int c = A.cur, k = threadIdx.x;
    cur_pose[k] = k < 9 ? M.R[9 * c + k] : k < 12 ? M.t[3 * c + k - 9] : k < 15 ? M.C[3 * c + k - 12]
                : k < 21 ? M.cam[6 * c + k - 15] : M.g_cs[c];
  }
  TV.pose = cur_pose;  // visible after the first barrier below
  const int K = M.kpkf_max;
  const int cur = A.cur;
  const int ncur = M.kp_n[cur], cur_off = M.kp_off[cur];
  const lm_fuse_cfg& fc = A.fc;
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  if (threadIdx.x < 16) tm[threadIdx.x] = 0;
  if (threadIdx.x == 0 && rank == 0) {
    M.scal[SC_DIRTY_N] = 0;  // k_fuse_refresh consumed the list
    nc_sh = 0;
    ni_sh = 0;
    nchg_sh = 0;
    tmin_sh = 0x7fffffff;
    s_nset = 0;
    tag_base = atomicAdd(&M.scal[SC_ROUND], T + 2);  // one dedupe tag per iteration (<= T + 1)
  }
  for (int t = threadIdx.x; t < T; t += REV_THREADS) {
    const int ts = M.s.targets[t];
    s_toff[t] = M.kp_off[ts];  // (every CTA: the helpers re-evaluate items too)
    if (rank == 0) {
      s_nact[t] = M.s.pinfo[PI_NACT * TMAX + t];
      s_live[t] = M.s.pinfo[PI_LIVE * TMAX + t];
      s_obs[t] = M.s.pinfo[PI_OBS * TMAX + t];
      M.s.pass_of[ts] = t;
    }
  }
  pair_acc_init<REV_THREADS>(&acc, A.cur);  // (barrier)
  const unsigned long long mpb = M.mp_rec_bytes;
  const unsigned long long ev_base = M.ledger[LG_SMALL_EVENTS];  // (the ledger changes only at the end)
  const int mtag = M.scal[SC_MTAG];
  // install point p's speculated post-ADD state (k_fuse_post): descriptor, geometry, hit
  auto install_post = [&](int p) {
    M.rep[2 * (size_t)p] = M.sp_rep[2 * (size_t)p];
    M.rep[2 * (size_t)p + 1] = M.sp_rep[2 * (size_t)p + 1];
    const double* sg = M.sp_geo + 5 * (size_t)p;
    M.gacc[3 * p] = sg[0];
    M.gacc[3 * p + 1] = sg[1];
    M.gacc[3 * p + 2] = sg[2];
    M.glo[p] = sg[3];
    M.ghi[p] = sg[4];
    M.gval[p] = 1;
    M.dirty[p] = 0;
    M.hit[p] = make_int2(M.ver[p], M.sp_hit[p]);
    hit_list_add(M, M.sp_hit[p], p);
    atomicAdd((unsigned long long*)&M.s.stats->dbg[12], 1ull);
  };
  const long long kf_cur = M.kf_id[A.cur];
  if (threadIdx.x == 0) tm[8] = gtime_p<P>() - t_entry;  // prologue
  long long alg = 0, npts = 0, nacts = 0, ledger_events = 0;
  int iter = 0, rounds = 0, pass_act = 0, reeval = 0, redo_pts = 0, mergeable = 0, touched_min = 0x7fffffff, fast_passes = 0;
  int t0 = 0;
  // append item (t, kp) to the re-evaluation list once per tag
  auto add_item = [&](int t, int kp, int tag) {
    const size_t it = (size_t)t * K + kp;
    if (atomicExch(&M.s.itag[it], tag) != tag) {
      const int at = atomicAdd(ni_p, 1);
      if (at < ILS) il_p[at] = (int)it;
      else M.s.ilist[at] = (int)it;
    }
  };
  auto passof = [&](int slot) -> int { return M.s.pass_of[slot]; };  // (read-only here: L1-resident)
  // items of point p (its current observations) in passes after t1; warp-cooperative; true
  // when p has one
  auto point_items = [&](int p, int t1, int tag) -> bool {
    const int lane = threadIdx.x & 31;
    const int2* o = M.obs + M.ooff[p];
    const int no = M.nobs[p];
    bool any = false;
    for (int e = lane; e < no; e += 32) {
      const int2 ob = o[e];
      const int tt = passof(ob.x);
      if (tt > t1) {
        add_item(tt, ob.y, tag);
        any = true;
      }
    }
    return __any_sync(0xffffffffu, any);
  };
  // eval_item(M, cur, t, targets[t], kp) with the pass's keypoint offset from shared memory and
  // the point's list offset loaded in the first round
  auto eval_rev = [&](int t, int kp) -> ItemVal {
    ItemVal v{-1, -3, 0, 0, ActRec{0, 0, 0, 0, 0}};
    const int mp = M.kbind[s_toff[t] + kp];
    if (mp < 0) return v;
    const int al = M.alive[mp], nob = M.nobs[mp], off = M.ooff[mp], j = M.hit[mp].y;
    if (!al) return v;
    v.mp = mp;
    v.nob = nob;
    v.j = j;
    if (j < 0) return v;
    atomicOr(&M.s.hitpass[j * HPW + (t >> 5)], 1u << (t & 31));
    const int owner = M.kbind[cur_off + j];
    // the first 16 list entries load with the owner (used if the keypoint is free: does the
    // point already observe the current keyframe?), later ones 16 at a time
    const int2* o = M.obs + off;
    int sl[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) sl[q] = q < nob ? o[q].x : -1;
    if (owner < 0) {
      bool f = false;
#pragma unroll
      for (int q = 0; q < 16; ++q) f |= sl[q] == cur;
      for (int k0 = 16; k0 < nob; k0 += 16) {
#pragma unroll
        for (int q = 0; q < 16; ++q) sl[q] = k0 + q < nob ? o[k0 + q].x : -1;
#pragma unroll
        for (int q = 0; q < 16; ++q) f |= sl[q] == cur;
      }
      if (!f) {
        v.a = ActRec{cur, mp, j, -1, LM_ACT_ADD};
        v.has = 1;
      }
    } else if (owner != mp && M.alive[owner]) {
      v.a = ActRec{cur, mp, j, owner, LM_ACT_MERGE};
      v.has = 1;
    }
    return v;
  };
  // link(M, p, cur, j, acc, fuse=true) of a direct-pass ADD, one warp: the lanes take the
  // covisibility bumps, lane 0 the record; every load is issued in the first rounds, before
  // any store (the keypoint level and the current keyframe's centre come from shared memory).
  // When the point's speculated post-ADD state (k_fuse_post) matches this ADD, the point takes
  // it at once (descriptor, geometry, hit) instead of the incremental geometry / stale flag.
  auto add_direct = [&](const ActRec x, int k, int t1, int tag) {
    const int lane = threadIdx.x & 31;
    const int p = x.pid, j = x.j;
    // first round: every scalar of the point, its speculated post-ADD state (used only when it
    // matches), the hit list count of j
    const int n = M.nobs[p], off = M.ooff[p], cap = M.ocap[p];
    const int dirty = M.dirty[p], gv = M.gval[p], vr = M.ver[p], found = M.found[p];
    const int lev = TV.lev[j];
    const int stag = M.sp_tag[p], sv0 = M.sp_ver0[p], sn0 = M.sp_nobs0[p], sj = M.sp_j[p];
    const double px = M.pos[3 * p], py = M.pos[3 * p + 1], pz = M.pos[3 * p + 2];
    const double lo = M.glo[p], hi = M.ghi[p];
    const double ax = M.gacc[3 * p], ay = M.gacc[3 * p + 1], az = M.gacc[3 * p + 2];
    int* cntp = M.counts + (size_t)p * M.L + lev;
    const int cv = *cntp;
    const double Sl = M.S[lev];
    const int hc = M.s.hl_cnt[j];
    const uint4 r0 = M.sp_rep[2 * (size_t)p], r1 = M.sp_rep[2 * (size_t)p + 1];
    const double* sg = M.sp_geo + 5 * (size_t)p;
    const double g0 = sg[0], g1 = sg[1], g2 = sg[2], g3 = sg[3], g4 = sg[4];
    const int sh_ = M.sp_hit[p];
    // second round: the observation entries, the hit list
    const int hp = lane < hc && lane < HL ? M.s.hl[j * HL + lane] : -1;
    const int2* o = M.obs + off;
    const int2 e0 = lane < n ? o[lane] : make_int2(cur, 0), e1 = lane + 32 < n ? o[lane + 32] : make_int2(cur, 0);
    const int o0 = e0.x, o1 = e1.x;
    const int last = n ? o[n - 1].x : -1;
    const bool spec = stag == mtag && sv0 == vr && sn0 == n && sj == j;
    // the record first (lane 0; its stores do not feed the item / hit-list walks below: the
    // point is already listed for this iteration, rmark == tag), so its chain overlaps theirs
    if (lane == 0) {
      int2* dst = M.obs + off;
      if (n == cap) {
        const int nc = cap < 4 ? 4 : 2 * cap;
        const int noff = atomicAdd(&M.scal[SC_OBS_HEAD], nc);
        if (noff + nc > M.obs_cap) {
          set_err(M, LM_ERR_CAPACITY);  // (the step fails; the record is left as it was)
          dst = nullptr;
        } else {
          copy_obs(M.obs + noff, o, n);
          M.ooff[p] = noff;
          M.ocap[p] = nc;
          dst = M.obs + noff;
        }
      }
      if (dst) {
        dst[n] = make_int2(cur, j);
        M.nobs[p] = n + 1;
        M.kbind[cur_off + j] = p;
        *cntp = cv + 1;
        M.ver[p] = vr + 1;
        M.found[p] = found + 1;
        if (spec) {
          M.rep[2 * (size_t)p] = r0;
          M.rep[2 * (size_t)p + 1] = r1;
          M.gacc[3 * p] = g0;
          M.gacc[3 * p + 1] = g1;
          M.gacc[3 * p + 2] = g2;
          M.glo[p] = g3;
          M.ghi[p] = g4;
          M.gval[p] = 1;
          M.dirty[p] = 0;
          M.hit[p] = make_int2(vr + 1, sh_);
          hit_list_add(M, sh_, p);
          atomicAdd((unsigned long long*)&M.s.stats->dbg[12], 1ull);
        } else {
          mark_dirty_owned(M, p, dirty);
          const long long kf_last = last >= 0 ? M.kf_id[last] : -1;
          if (gv && !dirty && (n == 0 || kf_last < kf_cur)) {
            const double rx = px - cur_pose[12], ry = py - cur_pose[13], rz = pz - cur_pose[14];
            const double dd = sqrt(rx * rx + ry * ry + rz * rz);
            if (dd > 0) {  // geo_term
              const double d0 = dd / Sl;
              M.glo[p] = d0 < lo ? d0 : lo;
              M.ghi[p] = d0 > hi ? d0 : hi;
              M.gacc[3 * p] = ax + rx / dd;
              M.gacc[3 * p + 1] = ay + ry / dd;
              M.gacc[3 * p + 2] = az + rz / dd;
            }
          } else {
            M.gval[p] = 0;
          }
        }
        inst_p[k] = spec;
        if (!spec) atomicAdd(nset_p, 1);
      }
    }
    // the point's items in passes after t1 (its observations after the ADD: the old ones and
    // (cur, j)), and the points hitting j (hit list): their hits are unchanged by the apply
    const int tt0 = passof(o0), tt1 = passof(o1), ttc = lane == 0 ? passof(cur) : -1;
    // hit-list point state in one round, its list head included (a point is listed under one
    // keypoint, its hit, so no other warp of this pass walks it; the action points are marked)
    const bool hv = hp >= 0;
    const int hal = hv ? M.alive[hp] : 0, hy = hv ? M.hit[hp].y : -2, hrm = hv ? M.s.rmark[hp] : tag;
    const int hno = hv ? M.nobs[hp] : 0, hof = hv ? M.ooff[hp] : 0;
    const bool hq = hv && hal && hy == j && hrm != tag;
    if (lane < n && tt0 > t1) add_item(tt0, e0.y, tag);
    if (lane + 32 < n && tt1 > t1) add_item(tt1, e1.y, tag);
    if (ttc > t1) add_item(ttc, j, tag);
    for (int e = lane + 64; e < n; e += 32) {
      const int2 ob = o[e];
      const int tt = passof(ob.x);
      if (tt > t1) add_item(tt, ob.y, tag);
    }
    unsigned hm = __ballot_sync(0xffffffffu, hq);
    while (hm) {  // hit-list points' items (their state is unchanged)
      const int src = __ffs(hm) - 1;
      hm &= hm - 1;
      const int qn = __shfl_sync(0xffffffffu, hno, src), qo = __shfl_sync(0xffffffffu, hof, src);
      for (int e = lane; e < qn; e += 32) {
        const int2 ob = M.obs[qo + e];
        const int tt = passof(ob.x);
        if (tt > t1) add_item(tt, ob.y, tag);
      }
    }
    if (hc > HL) {  // overflowed list: scan the passes of the keypoint's bitmap
      for (int w = 0; w < HPW; ++w) {
        unsigned bits = M.s.hitpass[j * HPW + w];
        while (bits) {
          const int tt = 32 * w + __ffs(bits) - 1;
          bits &= bits - 1;
          if (tt <= t1 || tt >= T) continue;
          const int nn = M.kp_n[M.s.targets[tt]];
          const int* pjt = M.s.pj + (size_t)tt * K;
          for (int kp = lane; kp < nn; kp += 32)
            if (pjt[kp] == j) add_item(tt, kp, tag);
        }
      }
    }
    covis_add(M, cur, o0, +1, &acc);
    covis_add(M, cur, o1, +1, &acc);
    for (int e = lane + 64; e < n; e += 32) covis_add(M, cur, o[e].x, +1, &acc);
    __syncwarp();
  };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // touched point p after the apply, one warp: its post-ADD state when the apply did exactly
  // the speculated ADD (same observation set as k_fuse_post's; the list is sorted: clean
  // before, the current keyframe appended last), else refresh (descriptor + geometry) and
  // a new hit
  auto settle_point = [&](int p) {
    if (M.sp_tag[p] == mtag && M.sp_ver0[p] >= 0 && M.ver[p] == M.sp_ver0[p] + 1 &&
        M.nobs[p] == M.sp_nobs0[p] + 1 && M.kbind[cur_off + M.sp_j[p]] == p) {
      if (lane == 0) install_post(p);
      __syncwarp();
      return;
    }
    if (M.dirty[p]) {
      refresh_rep_warp(M, p, lane);
      if (lane == 0) M.dirty[p] = 0;
      __syncwarp();
    }
    if (!M.gval[p]) geo_full_warp(M, p, lane);
    PGeo g;
    point_geometry(M, p, fc.dist_band_slack, g);  // (every lane: same loads, broadcast)
    const int j = gather_hit_warp(M, fc, g, cur, TV, lane);
    if (lane == 0) {
      M.hit[p] = make_int2(M.ver[p], j);
      hit_list_add(M, j, p);
    }
    __syncwarp();
  };
  // changed current keypoint q of a general pass: the points hitting it join the touched
  // list (hit list; a keypoint whose list overflowed scans the passes of its bitmap)
  auto hitlist_item = [&](int q, int t1, int tag) {
    const int k = M.s.chg[q];
    const int c = M.s.hl_cnt[k];
    if (c <= HL) {
      if (lane < c) {
        const int p = M.s.hl[k * HL + lane];
        if (M.alive[p] && M.hit[p].y == k && atomicExch(&M.s.rmark[p], tag) != tag)
          M.s.cands[atomicAdd(nc_p, 1)] = p;
      }
      return;
    }
    for (int w = 0; w < HPW; ++w) {
      unsigned bits = M.s.hitpass[k * HPW + w];
      while (bits) {
        const int tt = 32 * w + __ffs(bits) - 1;
        bits &= bits - 1;
        if (tt <= t1 || tt >= T) continue;
        const int n = M.kp_n[M.s.targets[tt]];
        const int* pjt = M.s.pj + (size_t)tt * K;
        for (int kp = lane; kp < n; kp += 32)
          if (pjt[kp] == k) add_item(tt, kp, tag);
      }
    }
  };
  // settle phase item k of a general pass: touched points (k < ncand) that have items in later
  // passes settle; the points hitting a re-bound keypoint list their items
  auto settle_item = [&](int k, int ncand, int t1, int tag) {
    const int p = M.s.cands[k];
    if (k < ncand) {
      if (!M.alive[p] || !M.s.cneed[k]) return;
      settle_point(p);
    } else {
      point_items(p, t1, tag);
    }
  };
  const int AW = (K + 31) >> 5;
  constexpr int RW = REV_THREADS / 32;  // warps per CTA
  // a phase goes to the whole cluster when its work exceeds this many rounds of CTA 0 alone
  // (byte 0: direct-pass actions; byte 1: the other phases; launch knob LM_REV_WIDE)
  const int wd = wide & 0xff, wo = (wide >> 8) & 0xff;
  // re-evaluation of listed item q: pass totals by deltas (CTA 0's counters), action bitmap
  // toggled
  auto rescan_item = [&](int q) {
    const int it = q < ILS ? il_p[q] : M.s.ilist[q];
    const int t = it / K, kp = it - t * K;
    const int oj = M.s.pj[it], ob = M.s.pob[it], oa = M.s.acts2[it].kind != 0;
    const ItemVal v = eval_rev(t, kp);
    store_item(M, it, v);
    const int dl = (v.mp >= 0) - (oj != -3), dob = v.nob - ob, da = v.has - oa;
    if (dl) atomicAdd(&live_p[t], dl);
    if (dob) atomicAdd(&obs_p[t], dob);
    if (da) {
      atomicAdd(&nact_p[t], da);
      atomicXor(&M.s.abits[(size_t)t * AW + (kp >> 5)], 1u << (kp & 31));
    }
    atomicMin(tmin_p, t);
  };
  if (rank > 0) {  // helper CTA: direct-pass actions k = rank*RW + wid (+ nranks*RW) on command
    for (;;) {
      cl.sync();  // (A) a command is published
      const int cmd = rcmd0[0];
      if (cmd == RC_EXIT) break;
      const int ht1 = rcmd0[1], htag = rcmd0[2], hna = rcmd0[3], hnc = rcmd0[4];
#ifdef LM_DIAG
      const long long hd0 = gtime_p<P>();
#endif
      if (cmd == RC_SETTLE) {
        for (int k = rank * RW + wid; k < hna; k += nranks * RW) settle_item(k, hnc, ht1, htag);
      } else if (cmd == RC_RESCAN) {
        for (int q = rank * REV_THREADS + threadIdx.x; q < hna; q += nranks * REV_THREADS) rescan_item(q);
      } else if (cmd == RC_HITLIST) {
        for (int q = rank * RW + wid; q < hna; q += nranks * RW) hitlist_item(q, ht1, htag);
      } else if (cmd == RC_PTITEMS) {
        for (int k = rank * RW + wid; k < hna; k += nranks * RW) {
          const bool later = point_items(M.s.cands[k], ht1, htag);
          if (hnc && lane == 0) M.s.cneed[k] = later;
        }
      } else {
        for (int k = rank * RW + wid; k < hna; k += nranks * RW) add_direct(M.s.acts[k], k, ht1, htag);
      }
#ifdef LM_DIAG
      if (lane == 0) atomicMax(&g_diag[60], (unsigned long long)(gtime_p<P>() - hd0));
#endif
      cl.sync();  // (B) this helper's actions are applied
    }
    pair_acc_flush<REV_THREADS>(M, &acc);
    cl.sync();  // (C) CTA 0's shared memory stays alive until every helper is done with it
    return;
  }  // words of a pass's action bitmap
  while (true) {
    // (1) warp 0: first pass (>= t0) with actions, ledger / byte accounting of the passes
    //     before it, that pass's actions in keypoint order (from its action bitmap), and the
    //     touched points (action points + current owners of the hit keypoints, deduplicated).
    //     The other warps snapshot the current keyframe's bindings.
    const long long ta = gtime_p<P>();
    if (wid == 1) {  // warp 1: the accounting (off warp 0's chain)
      int t1 = T;
      for (int tb = t0; tb < T; tb += 32) {
        const unsigned bal = __ballot_sync(0xffffffffu, tb + lane < T && s_nact[tb + lane] > 0);
        if (bal) {
          t1 = tb + __ffs(bal) - 1;
          break;
        }
      }
      const int te = t1 < T ? t1 : T - 1;
      long long a_b = 0, a_p = 0, a_n = 0;
      for (int t = t0 + lane; t <= te; t += 32) {
        a_b += pass_bytes(s_live[t], s_obs[t], ncur, s_nact[t]);
        a_p += s_live[t];
        a_n += s_nact[t];
      }
      for (int off = 16; off; off >>= 1) {
        a_b += __shfl_xor_sync(0xffffffffu, a_b, off);
        a_p += __shfl_xor_sync(0xffffffffu, a_p, off);
        a_n += __shfl_xor_sync(0xffffffffu, a_n, off);
      }
      alg += a_b;  // (meaningful on thread 32)
      npts += a_p;
      nacts += a_n;
      {  // one record_small_transfer per reverse pass, in pass order (after the forward one)
        const unsigned long long ev0 = ev_base;
        for (int t = t0 + lane; t <= te; t += 32)
          if (ev0 + t < (unsigned long long)LG_LOG_CAP) M.lg_log[ev0 + t] = (long long)s_live[t] * (long long)mpb;
      }
      ledger_events += te - t0 + 1;
    }
    if (wid == 0) {
      int t1 = T;
      for (int tb = t0; tb < T; tb += 32) {
        const unsigned bal = __ballot_sync(0xffffffffu, tb + lane < T && s_nact[tb + lane] > 0);
        if (bal) {
          t1 = tb + __ffs(bal) - 1;
          break;
        }
      }
      int na = 0;
      const int tg = tag_base + 1 + iter;
      if (t1 < T) {
        const unsigned* bits = M.s.abits + (size_t)t1 * AW;
        const ActRec* seg = M.s.acts2 + (size_t)t1 * K;
        if (AW <= 64) {
          // lane per word pair (w = lane, lane + 32): the word prefix counts give each action
          // its position (keypoint order = word order); the keypoint indices go to s_il (free
          // until this iteration's items are listed), then the records load lane-parallel, up
          // to four per lane in flight (a word with many actions no longer loads them in a
          // dependent chain on one lane)
          const unsigned b0 = lane < AW ? bits[lane] : 0u, b1 = lane + 32 < AW ? bits[lane + 32] : 0u;
          const int c0 = __popc(b0), c1 = __popc(b1);
#ifdef LM_DIAG
          if (lane == 0) g_diag[48] += gtime_p<P>() - ta;
#endif
          int p0 = c0, p1 = c1;
          for (int off = 1; off < 32; off <<= 1) {
            const int y0 = __shfl_up_sync(0xffffffffu, p0, off), y1 = __shfl_up_sync(0xffffffffu, p1, off);
            if (lane >= off) {
              p0 += y0;
              p1 += y1;
            }
          }
          const int tot0 = __shfl_sync(0xffffffffu, p0, 31);
          na = tot0 + __shfl_sync(0xffffffffu, p1, 31);
          const int pre0 = p0 - c0, pre1 = tot0 + p1 - c1;
          auto put = [&](int at, const ActRec& x) {
            const ActRec y{cur, x.pid, x.j, x.other, x.kind};
            if (at < DMAX) s_acts[at] = y;
            M.s.acts[at] = y;
          };
          if (na <= ILS) {
            int at = pre0;
            for (unsigned r = b0; r; r &= r - 1) s_il[at++] = 32 * lane + __ffs(r) - 1;
            at = pre1;
            for (unsigned r = b1; r; r &= r - 1) s_il[at++] = 32 * (lane + 32) + __ffs(r) - 1;
            __syncwarp();
            for (int k0 = 0; k0 < na; k0 += 128) {
              ActRec xr[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int k = k0 + 32 * i + lane;
                if (k < na) xr[i] = seg[s_il[k]];
              }
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int k = k0 + 32 * i + lane;
                if (k < na) put(k, xr[i]);
              }
            }
          } else {
            int at = pre0;
            for (unsigned r = b0; r; r &= r - 1) put(at++, seg[32 * lane + __ffs(r) - 1]);
            at = pre1;
            for (unsigned r = b1; r; r &= r - 1) put(at++, seg[32 * (lane + 32) + __ffs(r) - 1]);
          }
#ifdef LM_DIAG
          if (lane == 0) g_diag[49] += gtime_p<P>() - ta;
#endif
        } else for (int wb = 0; wb < AW; wb += 32) {
          const int w = wb + lane;
          unsigned bw = w < AW ? bits[w] : 0u;
          const int c = __popc(bw);
          int pre = c;
          for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pre, off);
            if (lane >= off) pre += y;
          }
          int at = na + pre - c;
          while (bw) {
            const int kp = 32 * w + __ffs(bw) - 1;
            bw &= bw - 1;
            const ActRec x = seg[kp];
            const ActRec y{cur, x.pid, x.j, x.other, x.kind};
            if (at < DMAX) s_acts[at] = y;
            M.s.acts[at++] = y;
          }
          na += __shfl_sync(0xffffffffu, pre, 31);
        }
        __syncwarp();
        // direct pass: every action a plain ADD of a distinct point into a distinct keypoint
        bool simple = na <= 32;
        if (simple) {
          const ActRec x = lane < na ? s_acts[lane] : ActRec{0, -1 - lane, -1 - lane, 0, LM_ACT_ADD};
          const unsigned mj = __match_any_sync(0xffffffffu, x.j), mp = __match_any_sync(0xffffffffu, x.pid);
          simple = __all_sync(0xffffffffu, x.kind == LM_ACT_ADD && __popc(mj) == 1 && __popc(mp) == 1);
        } else if (na <= DMAX && AW <= JBW) {
          // distinct keypoints by a bitmap (the points of one pass are distinct: the bound points
          // of one keyframe's keypoints)
          for (int w = lane; w < AW; w += 32) s_jb[w] = 0u;
          __syncwarp();
          bool ok = true;
          for (int k = lane; k < na; k += 32) {
            const ActRec x = s_acts[k];
            const unsigned b = 1u << (x.j & 31);
            ok &= x.kind == LM_ACT_ADD && !(atomicOr(&s_jb[x.j >> 5], b) & b);
          }
          simple = __all_sync(0xffffffffu, ok);
        }
        if (simple) {
          for (int k = lane; k < na; k += 32) {  // touched points: the action points
            const int p = s_acts[k].pid;
            M.s.rmark[p] = tg;
            M.s.cands[k] = p;
          }
          if (lane == 0) nc_sh = na;
        } else {
          for (int k = lane; k < na; k += 32) {
            const ActRec x = M.s.acts[k];
            const int cand[3] = {x.pid, x.other, M.kbind[cur_off + x.j]};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const int p = cand[c];
              if (p >= 0 && atomicExch(&M.s.rmark[p], tg) != tg) M.s.cands[atomicAdd(&nc_sh, 1)] = p;
            }
          }
        }
        if (lane == 0) fast_sh = simple;
      }
      if (lane == 0) {
        t1_sh = t1;
        na_sh = na;
        tag_sh = tg;
      }
#ifdef LM_DIAG
      if (lane == 0) g_diag[50] += gtime_p<P>() - ta;
#endif
    }
    __syncthreads();
#ifdef LM_DIAG
    if (threadIdx.x == 0) g_diag[51] += gtime_p<P>() - ta;
#endif
    if (threadIdx.x == 0) tm[1] += gtime_p<P>() - ta;
    const int t1 = t1_sh;
    if (t1 >= T) break;
    if (pass_act > 0) mergeable += touched_min > t1;
    ++pass_act;
    const int na = na_sh, tag = tag_sh, ncand = nc_sh;
    // items of point p (its current observations) in passes after t1; warp-cooperative
    auto add_point_items = [&](int p) -> bool { return point_items(p, t1, tag); };
    // points hitting current keypoint k, whose binding changed, join the touched list (hit
    // list; a keypoint whose list overflowed falls back to scanning the passes of its bitmap)
    if (fast_sh) {
      // every action a plain ADD of a distinct point into a distinct unbound keypoint (the
      // pass's item is current, so slot j is free and the point does not see the current
      // keyframe): the actions touch disjoint entities and commute; apply them directly, each
      // point taking its speculated post-ADD state at once. The changed current keypoints are
      // exactly the actions' keypoints, and an ADD only adds an observation, so the touched
      // items are the points' observations after the apply.
      // (8 lanes per action, four actions per warp, measured 5% slower on C2: more registers
      // spilled and the tile syncs; a warp per action stays)
      // the helper CTAs take their share of the actions when there are more than CTA 0 has
      // warps (a pass CTA 0 covers alone skips the two cluster barriers)
      const bool wide_d = nranks > 1 && na > RW * wd;
      if (wide_d) {
        if (threadIdx.x == 0) {
          rcmd[0] = RC_DIRECT;
          rcmd[1] = t1;
          rcmd[2] = tag;
          rcmd[3] = na;
        }
        cl.sync();  // (A)
      }
#ifdef LM_DIAG
      const long long hd0 = gtime_p<P>();
#endif
      for (int k = wid; k < na; k += wide_d ? nranks * RW : RW) add_direct(s_acts[k], k, t1, tag);
#ifdef LM_DIAG
      if (lane == 0) atomicMax(&g_diag[61], (unsigned long long)(gtime_p<P>() - hd0));
      if (threadIdx.x == 0) g_diag[52] += hd0 - ta;  // walk + command
#endif
      if (wide_d) cl.sync();  // (B)
      __syncthreads();
#ifdef LM_DIAG
      if (threadIdx.x == 0) {
        g_diag[53] += gtime_p<P>() - hd0;  // direct apply wall
        g_diag[54] += g_diag[60] > g_diag[61] ? g_diag[60] : g_diag[61];  // slowest add_direct
        g_diag[55] += g_diag[61];
        g_diag[60] = g_diag[61] = 0;
        g_diag[56] += 1;
        g_diag[57] += na;
      }
#endif
      if (threadIdx.x == 0) {
        cnt[1] += na;
        ++rounds;
        ++fast_passes;
        tm[7] += gtime_p<P>() - ta;
        tm[2] += gtime_p<P>() - ta;
      }
      redo_pts += ncand;
      if (s_nset) {  // points whose speculated state did not apply: refresh + new hit
        const long long tv = gtime_p<P>();
        for (int k = wid; k < na; k += REV_THREADS / 32)
          if (!s_inst[k]) settle_point(s_acts[k].pid);
        __syncthreads();
        if (threadIdx.x == 0) tm[0] += gtime_p<P>() - tv;
      }
    } else {
      // the touched points' items before the apply (more points than CTA 0 has warps: on the
      // whole cluster), the current keyframe's bindings before
      const bool wide_p = nranks > 1 && ncand > RW * wo;
      auto command_items = [&](int cneed) {
        if (threadIdx.x == 0) {
          rcmd[0] = RC_PTITEMS;
          rcmd[1] = t1;
          rcmd[2] = tag;
          rcmd[3] = ncand;
          rcmd[4] = cneed;
        }
        cl.sync();  // (A)
      };
      if (wide_p) command_items(0);
      for (int k = wid; k < ncand; k += wide_p ? nranks * RW : RW) add_point_items(M.s.cands[k]);
      for (int k = threadIdx.x; k < ncur; k += REV_THREADS) M.s.snap[k] = M.kbind[cur_off + k];  // bindings before
      if (wide_p) cl.sync();  // (B)
      __syncthreads();
      if (threadIdx.x == 0) tm[7] += gtime_p<P>() - ta;
      rounds += apply_block<REV_THREADS, P>(M, M.s.acts, na, cnt, sh, &acc, tm);  // (barriers)
    if (threadIdx.x == 0) tm[2] += gtime_p<P>() - ta;
    // (2) after the apply: the touched points' items, and the points hitting a current
    //     keypoint whose binding changed (hit list; a keypoint whose list overflowed falls
    //     back to scanning the passes of its bitmap) join the touched list
    const long long tv = gtime_p<P>();
    if (wide_p) command_items(1);
    for (int k = wid; k < ncand; k += wide_p ? nranks * RW : RW) {
      const bool later = add_point_items(M.s.cands[k]);
      if (lane == 0) M.s.cneed[k] = later;  // no later item: its new hit is not needed this step
    }
    for (int k = threadIdx.x; k < ncur; k += REV_THREADS)  // current keypoints whose binding changed
      if (M.kbind[cur_off + k] != M.s.snap[k]) M.s.chg[atomicAdd(&nchg_sh, 1)] = k;
    if (wide_p) cl.sync();  // (B)
    __syncthreads();
    if (threadIdx.x == 0) tm[4] += gtime_p<P>() - tv;
    const long long tv2 = gtime_p<P>();
    const int nchg = nchg_sh;
    const bool wide_h = nranks > 1 && nchg > RW * wo;
    if (wide_h) {
      if (threadIdx.x == 0) {
        rcmd[0] = RC_HITLIST;
        rcmd[1] = t1;
        rcmd[2] = tag;
        rcmd[3] = nchg;
      }
      cl.sync();  // (A)
    }
    for (int q = wid; q < nchg; q += wide_h ? nranks * RW : RW) hitlist_item(q, t1, tag);
    if (wide_h) cl.sync();  // (B)
    __syncthreads();
    if (threadIdx.x == 0) tm[5] += gtime_p<P>() - tv2;
    const long long tv3 = gtime_p<P>();
    // (3) touched points, warp each: refresh (descriptor + geometry) where stale, then the new
    //     hit (lane 0); the hit-list points' items (their state is unchanged)
    // (a touched point without items in later passes keeps its dirty flag -- the next step's
    //  refresh picks it up -- and a stale hit: nothing reads it, the version differs). More
    //  points than CTA 0 has warps go to the whole cluster (the helper CTAs on command).
    const int nall = nc_sh;
    redo_pts += ncand;
    const bool wide = nranks > 1 && nall > RW * wo;
    if (wide) {
      if (threadIdx.x == 0) {
        rcmd[0] = RC_SETTLE;
        rcmd[1] = t1;
        rcmd[2] = tag;
        rcmd[3] = nall;
        rcmd[4] = ncand;
      }
      cl.sync();  // (A)
    }
    for (int k = wid; k < nall; k += wide ? nranks * RW : RW) settle_item(k, ncand, t1, tag);
    if (wide) cl.sync();  // (B)
    __syncthreads();
    if (threadIdx.x == 0) {
      tm[0] += gtime_p<P>() - tv;
      tm[6] += gtime_p<P>() - tv3;
    }
    }  // general path
    // (5) re-evaluate the listed items; pass totals by deltas, action bitmaps toggled
    const long long t7 = gtime_p<P>();
    const int ni = ni_sh;
    reeval += ni;
#ifdef LM_DIAG
    if (threadIdx.x == 0) {
      g_diag[58] += ni;
      g_diag[59] += 1;
    }
#endif
    // more items than CTA 0 has threads go to the whole cluster (the helpers on command)
    const bool wide_r = nranks > 1 && ni > REV_THREADS * wo;
    if (wide_r) {
      if (threadIdx.x == 0) {
        rcmd[0] = RC_RESCAN;
        rcmd[1] = t1;
        rcmd[2] = tag;
        rcmd[3] = ni;
      }
      cl.sync();  // (A)
    }
    for (int q = threadIdx.x; q < ni; q += wide_r ? nranks * REV_THREADS : REV_THREADS) rescan_item(q);
    if (wide_r) cl.sync();  // (B)
    __syncthreads();
    if (threadIdx.x == 0) {
      touched_min = tmin_sh;  // (diagnostic, thread 0's only: read here, before the reset below)
      tm[3] += gtime_p<P>() - t7;
      nc_sh = 0;  // counters of the next iteration (read above, before this barrier)
      ni_sh = 0;
      nchg_sh = 0;
      tmin_sh = 0x7fffffff;
      s_nset = 0;
    }
    t0 = t1 + 1;
    ++iter;
  }
  if (nranks > 1) {
    if (threadIdx.x == 0) rcmd[0] = RC_EXIT;
    cl.sync();  // (A) helpers leave their loop
  }
  __shared__ long long s_acct[4];  // warp 1's accounting, for thread 0's statistics below
  if (threadIdx.x == 32) {
    s_acct[0] = alg;
    s_acct[1] = npts;
    s_acct[2] = nacts;
    s_acct[3] = ledger_events;
  }
  pair_acc_flush<REV_THREADS>(M, &acc);  // (barriers)
  alg = s_acct[0];
  npts = s_acct[1];
  nacts = s_acct[2];
  ledger_events = s_acct[3];
  for (int t = threadIdx.x; t < T; t += REV_THREADS) M.s.pass_of[M.s.targets[t]] = -1;
  if (threadIdx.x == 0) {
    M.ledger[LG_NAIVE] += npts * mpb;  // record_small_transfer per pass (devicestore.py:94-101)
    M.ledger[LG_PERSIST] += npts * mpb;
    M.ledger[LG_SMALL_FUSE] += npts * mpb;
    M.ledger[LG_SMALL_EVENTS] += ledger_events;
    lm_step_stats* st = M.s.stats;
    st->merged += cnt[0];
    st->observations_added += cnt[1];
    st->stale += cnt[2];
    st->fuse_bytes += alg;
    st->fuse_bytes_rev += alg;
    st->fuse_passes += T;
    st->fuse_points += npts;
    st->fuse_actions += nacts;
    st->apply_rounds += rounds;
    st->fuse_cycles[4] += tm[0];
    st->fuse_cycles[5] += tm[1];
    st->fuse_cycles[6] += tm[2];
    st->fuse_cycles[7] += tm[3];
    for (int k = 8; k < 13; ++k) st->fuse_cycles[k] += tm[k];
    st->fuse_cycles[1] += redo_pts;  // touched points recomputed (count, not ns)
    st->rev_passes_acting += pass_act;
    st->rev_passes_redo += reeval;   // re-evaluated items (count)
    st->rev_mergeable += mergeable;
    for (int k = 4; k < 8; ++k) st->dbg[k] += tm[k];
    st->dbg[0] += fast_passes;  // diagnostics: acting passes applied directly (all plain ADDs)
  }
  if (nranks > 1) cl.sync();  // (C) the helpers are done with this CTA's shared memory
}

// deferred visible counters of every reverse pass (thread per item); a point merged away
// later in this step's reverse phase passes its bump on to its winner
__device__ __forceinline__ void visible_item(const DevMap& M, const StepArgs& A) {
  if (!A.do_fuse) return;
  const int t = blockIdx.y;
  if (t >= M.s.fctl[FC_T]) return;
  const int n = M.kp_n[M.s.targets[t]];
  const int kp = blockIdx.x * 256 + threadIdx.x;
  if (kp >= n) return;
  const size_t it = (size_t)t * M.kpkf_max + kp;
  if (M.s.pj[it] < -1) return;
  int p = M.s.pmp[it];
  const int tag = M.scal[SC_MTAG];
  for (int hop = 0; hop < 1 << 20 && !M.alive[p]; ++hop) {
    const int2 m = M.mrg[p];
    if (m.x != tag) break;
    p = m.y;
  }
  atomicAdd(&M.visible[p], 1);
}

}  // namespace lm
