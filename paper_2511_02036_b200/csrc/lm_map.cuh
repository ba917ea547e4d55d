// lm_map.cuh -- device-resident map store and its mutation primitives.
//
// Layout (all arenas allocated once per map, SoA, indexed by keyframe slot / global
// keypoint index / map point id):
//   keyframes  kf_id, state, kp_off, kp_n, q[4], R[9], t[3], C[3], P[12], cam[6], cell grid
//   keypoints  u, v (f64), level (u8), desc (2 x uint4), binding (i32, -1 = unbound)
//   points     pos[3] (f64), rep (2 x uint4), alive, found, visible, first_kf,
//              observation list (slot, kp) in an 8-byte pool, sorted by keyframe id,
//              per-level counters counts[id*L + level]
//   covis      dense int32 [kf_cap x kf_cap], symmetric
//
// The primitives restate MapModel's bookkeeping (pkg/src/localmap/mapmodel.py):
//   link        _record_obs 150-155        unlink_at   _unrecord_obs 157-163
//   kill_point  kill_map_point 233-237     replace     replace_map_point 245-267
//   merge_pair  fusion._merge 295-304      refresh     _refresh_rep_descriptor 165-181
// Covisibility updates are atomicAdd (commutative, order-free); everything else is
// single-writer per entity. The representative descriptor is refreshed lazily: the
// reference recomputes it after every observation change, but it is a pure function of
// the observation list and is only read by the fusion gather and by export, so
// mutations mark the point dirty and `refresh_dirty` recomputes it before those reads.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lm_b200.h"

namespace lm {

constexpr int NMAX = LM_MAX_NEIGHBORS;  // neighbours per triangulation step
constexpr int TMAX = LM_MAX_TARGETS;    // fusion targets per keyframe
constexpr int LMAX = 16;                // pyramid levels
constexpr int GRID_CELLS = 4096;        // cells per keyframe grid
constexpr int REFRESH_MAXN = 512;       // observations handled by the rep-refresh fast path
constexpr int MATCH_TILE = 32;          // current keypoints per match CTA (one per lane)
#ifndef LM_MATCH_WARPS
#define LM_MATCH_WARPS 8
#endif
constexpr int MATCH_WARPS = LM_MATCH_WARPS;  // warps per match CTA, each scanning a slice of j
constexpr int MATCH_JT = 1024;          // neighbour descriptors staged per smem chunk
constexpr int RES_PAIR = 1 << 20;       // hashed (point, keyframe) reservation keys per map
constexpr int HL = 16;                  // hit-list entries per current keypoint
constexpr int LG_LOG_CAP = 1 << 16;     // logged small-transfer events per map

enum KfState { KF_FREE = 0, KF_STAGED = 1, KF_LIVE = 2, KF_DEAD = 3 };
// SC_ERR: sticky (arena overflow: the map is unusable); SC_SOFT: this step's recoverable
// contract error (a stage touched a non-resident keyframe), cleared at every step start
// SC_NORES: 1 = the stages do not enforce residency (the caller's store is not this map's)
enum Scal { SC_NEXT_ID = 0, SC_OBS_HEAD, SC_RECENT_N, SC_ERR, SC_DIRTY_N, SC_ROUND, SC_MTAG, SC_SOFT, SC_NORES,
            SC_N = 16 };
enum LedgerIdx { LG_PERSIST = 0, LG_NAIVE, LG_SMALL_TRI, LG_SMALL_FUSE, LG_SMALL_EVENTS, LG_EVICT, LG_N = 8 };
enum CandStatus { CS_PASS = 0, CS_PARALLAX = 1, CS_DEPTH = 2, CS_REPROJ = 3, CS_SCALE = 4, CS_DEGEN = 5 };

struct ActRec {  // gathered fusion action (device form)
  int slot;      // target keyframe slot
  int pid;       // projected point
  int j;         // keypoint hit
  int other;     // existing point (MERGE) or -1
  int kind;      // LM_ACT_ADD / LM_ACT_MERGE
};

struct PGeo {  // _point_geometry row (fusion.py:57-94)
  double x, y, z, blo, bhi, d0, vx, vy, vz;
  uint4 r0, r1;
  int ok;
};

// per-step scratch of one map
struct Scratch {
  // triangulation
  int n_nbr;
  int* nbr;              // [NMAX] slots
  int* deg;              // [NMAX]
  double* F;             // [NMAX*9]
  int* cur_sorted;       // [kpkf_max]
  int* cur_bucket;       // [LMAX+1]
  int* tiles;            // [(kpkf_max/MATCH_TILE + LMAX) * 3] level,start,count
  int* n_tiles;          // [1]
  int* nb_n;             // [NMAX]
  int* nb_bucket;        // [NMAX*(LMAX+1)]
  int* nb_j;             // [NMAX*kpkf_max]
  uint4* nb_desc;        // [NMAX*kpkf_max*2]
  double* nb_u;          // [NMAX*kpkf_max]
  double* nb_v;
  double* nb_thr;
  unsigned long long* pick;   // [NMAX*kpkf_max] (dist<<32 | j)
  unsigned long long* bestj;  // [NMAX*kpkf_max] (dist<<32 | i)
  int* cand_n;           // [NMAX]
  int* cand_i;           // [NMAX*kpkf_max]
  int* cand_j;
  int* cand_d;
  int* cand_st;
  double* cand_X;        // [NMAX*kpkf_max*3]
  int* win_rank;         // [kpkf_max]
  int* crank;            // [NMAX*kpkf_max] creation rank of a candidate (-1: not created)
  int* cmeta;            // [4] first new id, observation head, probation length at commit
  unsigned char* mask_cur;  // optional explicit unbound masks (lm_search)
  unsigned char* mask_nbr;
  // fusion
  int* targets;          // [TMAX]
  int* n_targets;        // [1]
  int* rank_buf;         // [TMAX * kf_cap] second-order walk scratch
  int* pts;              // [max(kpkf_max, pts_cap)] point list of the current pass
  int* pend;             // [act_cap] pending action indices (apply rounds)
  int* merge_a;          // [act_cap] merges committed this round (warp-cooperative)
  int* merge_b;
  int* ready;            // [act_cap]
  PGeo* geo;             // [pts_cap]
  ActRec* acts;          // [TMAX*kpkf_max]
  ActRec* acts2;         // [TMAX*kpkf_max] forward gather output, per-CTA segments
  int* blk_cnt;          // [act_cap/256 + 1]
  int* blk_off;
  int* fctl;             // [8] fusion control: targets, forward points, ...
  int* pass_j;           // [kpkf_max] per-pass resolved hit per target keypoint
  int* add_list;         // [act_cap] high-degree ADDs committed warp-cooperatively
  int* def;              // [act_cap] ready ADDs of this round (grouped per point)
  unsigned long long* dnxt;  // [act_cap] ticket of a ready ADD within its point's group
  int* gbase;            // [mp_cap] observation-list position of a group's first new entry
  // reverse passes
  int* pinfo;            // [3*TMAX] per pass: actions, live bound points, observation sum
  unsigned* hitpass;     // [kpkf_max*HPW] per current keypoint: bitmap of passes hitting it
  int* pj;               // [TMAX*kpkf_max] per (pass, keypoint): resolved hit (-3 not bound)
  int* pass_of;          // [kf_cap] keyframe slot -> pass index (-1)
  int* snap;             // [kpkf_max] current keyframe bindings before an apply
  int* chg;              // [kpkf_max] current keypoints whose binding an apply changed
  int* rmark;            // [mp_cap] dedup tag of the touched-point list
  int* die;              // [mp_cap] apply round (tag) in which the point loses a merge
  int* pmp;              // [TMAX*kpkf_max] per (pass, keypoint): bound live point at evaluation
  int* pob;              // [TMAX*kpkf_max] per (pass, keypoint): its observation count then
  int* itag;             // [TMAX*kpkf_max] dedup tag of the re-evaluation list
  int* ilist;            // [TMAX*kpkf_max] (pass, keypoint) items to re-evaluate
  int* cands;            // [act_cap] points touched by an apply
  int* cneed;            // [act_cap] touched point has items in later passes
  int* hl_cnt;           // [kpkf_max] per current keypoint: points whose hit is it (count)
  int* hl;               // [kpkf_max*HL] ... (ids; entries whose hit moved are skipped)
  int* hreg;             // [mp_cap] step tag: point already listed by the speculative scan
  int* upts;             // [act_cap] distinct bound points of all reverse passes
  int* sp_list;          // [act_cap] points with a speculative reverse-pass ADD
  int2* sp_obs;          // [POST_BLOCKS*8*(POST_MAXN+1)] per-warp virtual observation lists
  unsigned* abits;       // [TMAX*ceil(kpkf_max/32)] per pass: keypoints whose item has an action
  int* act_flag;         // [TMAX*kpkf_max]
  int* vis_flag;         // [TMAX*kpkf_max]
  int pts_cap;
  int act_cap;
  lm_step_stats* stats;  // [1]
};

struct DevMap {
  int kf_cap, kp_cap, kpkf_max, mp_cap, obs_cap, L, min_w, min_obs_keep, recent_cap;
  int kp_rec_bytes, desc_bytes, mp_rec_bytes;
  double sf, log_sf;
  double S[LMAX], S2[LMAX];
  // keyframes
  long long* kf_id;
  int* kf_state;
  unsigned char* kf_res;  // DeviceStore residency (devicestore.py:62-78): 1 after upload, 0 after evict
  int* kp_off;
  int* kp_n;
  double* q;
  double* R;
  double* t;
  double* C;
  double* P;
  double* cam;
  double* g_cs;
  int* g_nx;
  int* g_ny;
  int* cell_start;  // [kf_cap*(GRID_CELLS+1)]
  int* cell_items;  // [kp_cap] global keypoint index
  // keypoints
  double* ku;
  double* kv;
  unsigned char* klev;
  uint4* kdesc;
  int* kbind;
  // points
  double* pos;
  uint4* rep;
  unsigned char* alive;
  int* found;
  int* visible;
  long long* first_kf;
  int* nobs;
  int* ocap;
  int* ooff;
  int2* obs;
  int* counts;
  int* dirty;        // representative descriptor + geometry cache stale
  int* dirty_list;   // ids whose dirty flag went 0 -> 1 (SC_DIRTY_N entries)
  // per-point view-geometry cache (fusion.py:57-94 accumulators over the sorted
  // observations): sum of unit rays, min/max level-0 distance, valid flag
  double* gacc;      // [mp_cap*3]
  double* glo;
  double* ghi;
  unsigned char* gval;
  int* ver;          // bumped on every observation change (speculative reverse gather)
  int2* mrg;         // loser -> {merge tag, winner}: deferred visible bumps follow it (SC_MTAG)
  // speculative post-ADD state of points with a reverse-pass ADD (k_fuse_post), valid when
  // sp_tag == SC_MTAG and the point changed exactly by that ADD
  int* sp_tag;
  int* sp_j;
  int* sp_ver0;
  int* sp_nobs0;
  int* sp_hit;
  uint4* sp_rep;     // [mp_cap*2]
  double* sp_geo;    // [mp_cap*5] gacc xyz, lo, hi
  int2* hit;         // per point: {version, hit into the current keyframe (-2/-1/j)}
  // deterministic-reservation tables (apply): round-tagged min action index per entity
  unsigned long long* res_pt;    // [mp_cap]
  unsigned long long* res_slot;  // [kp_cap]
  unsigned long long* res_ex;    // [mp_cap] min tag of the actions that need the point exclusively
  unsigned long long* res_pair;  // [RES_PAIR] (point, keyframe) ADD keys, hashed (collisions only serialise)
  unsigned long long* grp_head;  // [mp_cap] ready ADDs of the point this round: (round << 32 | count)
  // covisibility
  int* covis;
  // probation list (culling.RecentPoint)
  int* recent_id;
  int* recent_born;
  // scalars
  int* scal;
  unsigned long long* ledger;
  // per_stage_small_transfers (devicestore.py:94-101): bytes of every record_small_transfer
  // event in order (all are "fusion": one forward pass + one per reverse pass), entry k =
  // event k; events past LG_LOG_CAP keep counting in the ledger totals only
  long long* lg_log;
  Scratch s;
};

__device__ __forceinline__ void set_err(const DevMap& M, int code) { atomicCAS(&M.scal[SC_ERR], 0, code); }

__device__ __forceinline__ int hamming(uint4 a0, uint4 a1, uint4 b0, uint4 b1) {
  return __popc(a0.x ^ b0.x) + __popc(a0.y ^ b0.y) + __popc(a0.z ^ b0.z) + __popc(a0.w ^ b0.w) +
         __popc(a1.x ^ b1.x) + __popc(a1.y ^ b1.y) + __popc(a1.z ^ b1.z) + __popc(a1.w ^ b1.w);
}

// Shared-memory accumulator of covisibility deltas: the commutative bumps of a whole
// kernel land in shared memory (one smem atomic each) and are flushed to the dense matrix
// once, instead of contending global atomics on a few hot pairs. Pairs of keyframes in the
// window of the PAIR_W most recent slots use a dense upper-triangle table (no probing);
// other pairs an open-addressing hash; overflow falls back to global atomics.
constexpr int PAIR_W = 96;
constexpr int PAIR_T = PAIR_W * (PAIR_W - 1) / 2;
constexpr int PAIR_H = 1024;
struct PairAcc {
  int wbase;
  int win[PAIR_T];
  unsigned key[PAIR_H];  // lo << 16 | hi, 0xffffffff = empty
  int val[PAIR_H];
};

__device__ __forceinline__ void covis_global(const DevMap& M, int a, int b, int d) {
  atomicAdd(&M.covis[(size_t)a * M.kf_cap + b], d);
  atomicAdd(&M.covis[(size_t)b * M.kf_cap + a], d);
}

__device__ __forceinline__ int tri_index(int i, int j) {  // i < j < PAIR_W
  return i * (2 * PAIR_W - i - 1) / 2 + (j - i - 1);
}

__device__ __forceinline__ void covis_add(const DevMap& M, int a, int b, int d, PairAcc* acc = nullptr) {
  if (a == b) return;
  if (acc) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    const int il = lo - acc->wbase, ih = hi - acc->wbase;
    if (il >= 0 && ih < PAIR_W) {
      atomicAdd(&acc->win[tri_index(il, ih)], d);
      return;
    }
    const unsigned k = (unsigned)lo << 16 | (unsigned)hi;
    unsigned h = (k * 2654435761u) >> 22;  // 10 bits
    for (int probe = 0; probe < 16; ++probe) {
      const unsigned cur = acc->key[h];
      if (cur == k) {
        atomicAdd(&acc->val[h], d);
        return;
      }
      if (cur == 0xffffffffu) {
        const unsigned prev = atomicCAS(&acc->key[h], 0xffffffffu, k);
        if (prev == 0xffffffffu || prev == k) {
          atomicAdd(&acc->val[h], d);
          return;
        }
      }
      h = (h + 1) & (PAIR_H - 1);
    }
  }
  covis_global(M, a, b, d);
}

// covisibility delta d between keyframe `slot` and every observer of o[0..n): the list
// entries are loaded 8 at a time before their atomics (one L2 round trip per 8 entries
// instead of one per entry: the compiler does not hoist loads across the atomics)
__device__ __forceinline__ void covis_list(const DevMap& M, int slot, const int2* o, int n, int d, PairAcc* acc) {
  int s[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] = j < n ? o[j].x : slot;
  for (int k0 = 0; k0 < n; k0 += 8) {
    int nx[8];  // the next chunk's loads are in flight while this chunk's bumps run
#pragma unroll
    for (int j = 0; j < 8; ++j) nx[j] = k0 + 8 + j < n ? o[k0 + 8 + j].x : slot;
#pragma unroll
    for (int j = 0; j < 8; ++j) covis_add(M, slot, s[j], d, acc);  // (slot, slot) is a no-op
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = nx[j];
  }
}

template <int BLOCK>
__device__ void pair_acc_init(PairAcc* acc, int newest_slot) {
  for (int q = threadIdx.x; q < PAIR_T; q += BLOCK) acc->win[q] = 0;
  for (int h = threadIdx.x; h < PAIR_H; h += BLOCK) {
    acc->key[h] = 0xffffffffu;
    acc->val[h] = 0;
  }
  if (threadIdx.x == 0) acc->wbase = newest_slot - (PAIR_W - 1) < 0 ? 0 : newest_slot - (PAIR_W - 1);
  __syncthreads();
}

template <int BLOCK>
__device__ void pair_acc_flush(const DevMap& M, PairAcc* acc) {
  __syncthreads();
  for (int q = threadIdx.x; q < PAIR_W * PAIR_W; q += BLOCK) {
    const int i = q / PAIR_W, j = q - i * PAIR_W;
    if (i < j) {
      const int v = acc->win[tri_index(i, j)];
      if (v) covis_global(M, acc->wbase + i, acc->wbase + j, v);
    }
  }
  for (int h = threadIdx.x; h < PAIR_H; h += BLOCK) {
    const unsigned k = acc->key[h];
    if (k != 0xffffffffu && acc->val[h] != 0) covis_global(M, (int)(k >> 16), (int)(k & 0xffff), acc->val[h]);
  }
  __syncthreads();
}

// copy n observation entries (8 loads in flight before their stores: source and
// destination are the same pool, so the compiler will not overlap them on its own)
__device__ __forceinline__ void copy_obs(int2* dst, const int2* src, int n) {
  for (int k0 = 0; k0 < n; k0 += 8) {
    int2 e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (k0 + j < n) e[j] = src[k0 + j];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (k0 + j < n) dst[k0 + j] = e[j];
  }
}

__device__ __forceinline__ int obs_find(const DevMap& M, int mp, int slot) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  if (n && o[n - 1].x == slot) return n - 1;  // the newest keyframe sorts last
  for (int k = 0; k < n; ++k)
    if (o[k].x == slot) return k;
  return -1;
}

// append (slot, kp); grows by doubling. Lists are kept sorted by keyframe id only while the
// point is clean: mutations append and mark the point dirty, and refresh_rep_warp sorts
// before anything order-dependent reads the list (invariant: clean => sorted).
// Returns the position, or -1 when the pool is exhausted.
__device__ int obs_insert(const DevMap& M, int mp, int slot, int kp) {
  const int n = M.nobs[mp];
  if (n == M.ocap[mp]) {
    const int nc = M.ocap[mp] < 4 ? 4 : 2 * M.ocap[mp];
    const int off = atomicAdd(&M.scal[SC_OBS_HEAD], nc);
    if (off + nc > M.obs_cap) {
      set_err(M, LM_ERR_CAPACITY);
      return -1;
    }
    const int2* src = M.obs + M.ooff[mp];
    copy_obs(M.obs + off, src, n);
    M.ooff[mp] = off;
    M.ocap[mp] = nc;
  }
  M.obs[M.ooff[mp] + n] = make_int2(slot, kp);
  M.nobs[mp] = n + 1;
  return n;
}

// does point mp observe keyframe slot? (branch-free scan, 16 independent loads in flight)
__device__ __forceinline__ bool observes(const DevMap& M, int mp, int slot) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  bool f = false;
  for (int k0 = 0; k0 < n; k0 += 16) {
    int s[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j] = k0 + j < n ? o[k0 + j].x : -1;
#pragma unroll
    for (int j = 0; j < 16; ++j) f |= s[j] == slot;
  }
  return f;
}

// the representative descriptor is stale until refreshed (rep is a pure function of the
// observation list; read only by the fusion gather and export)
__device__ __forceinline__ void mark_dirty(const DevMap& M, int mp) {
  if (atomicExch(&M.dirty[mp], 1) == 0) {
    const int at = atomicAdd(&M.scal[SC_DIRTY_N], 1);
    if (at < M.mp_cap) M.dirty_list[at] = mp;
  }
}

// mark_dirty for a caller that is the only one touching mp's flag in this phase and already
// read it (`was`): one returning atomic instead of two
__device__ __forceinline__ void mark_dirty_owned(const DevMap& M, int mp, int was) {
  if (was) return;
  M.dirty[mp] = 1;
  const int at = atomicAdd(&M.scal[SC_DIRTY_N], 1);
  if (at < M.mp_cap) M.dirty_list[at] = mp;
}

// one observation's contribution to the view geometry (fusion.py:77-84); false if skipped
__device__ __forceinline__ bool geo_term(const DevMap& M, int mp, int2 e, double& rx, double& ry, double& rz,
                                        double& dd, double& d0) {
  const int s = e.x;
  rx = M.pos[3 * mp] - M.C[3 * s];
  ry = M.pos[3 * mp + 1] - M.C[3 * s + 1];
  rz = M.pos[3 * mp + 2] - M.C[3 * s + 2];
  dd = sqrt(rx * rx + ry * ry + rz * rz);
  if (!(dd > 0)) return false;
  d0 = dd / M.S[M.klev[M.kp_off[s] + e.y]];
  return true;
}

// full recompute of the cache over the sorted observation list (sequential order = the
// reference's accumulation order, so the sums are bit-identical)
__device__ void geo_full(const DevMap& M, int mp) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  double lo = INFINITY, hi = -INFINITY, ax = 0, ay = 0, az = 0;
  for (int k = 0; k < n; ++k) {
    double rx, ry, rz, dd, d0;
    if (!geo_term(M, mp, o[k], rx, ry, rz, dd, d0)) continue;
    lo = d0 < lo ? d0 : lo;
    hi = d0 > hi ? d0 : hi;
    ax = ax + rx / dd;
    ay = ay + ry / dd;
    az = az + rz / dd;
  }
  M.gacc[3 * mp] = ax;
  M.gacc[3 * mp + 1] = ay;
  M.gacc[3 * mp + 2] = az;
  M.glo[mp] = lo;
  M.ghi[mp] = hi;
  M.gval[mp] = 1;
}

// _record_obs: covis +1 with every current observer, bind the slot, count the level. An
// observation appended after every existing one extends the cached sums exactly.
// Latency-shaped: the independent loads are issued together before any store.
// fuse=true: fusion's ADD_OBSERVATION on top (found += 1, representative descriptor marked
// stale), with the flag/counter loads in the same first round.
__device__ void link(const DevMap& M, int mp, int slot, int kp, PairAcc* acc = nullptr, bool fuse = false,
                     bool covis = true) {
  // every load first: the stores below would otherwise serialise them (aliasing)
  const int n = M.nobs[mp], cap = M.ocap[mp], off = M.ooff[mp];
  const int dirty = M.dirty[mp], gv = M.gval[mp], vr = M.ver[mp];
  const int found = fuse ? M.found[mp] : 0;
  const int g = M.kp_off[slot] + kp;
  const long long kf_new = M.kf_id[slot];
  const double px = M.pos[3 * mp], py = M.pos[3 * mp + 1], pz = M.pos[3 * mp + 2];
  const double cx = M.C[3 * slot], cy = M.C[3 * slot + 1], cz = M.C[3 * slot + 2];
  const double lo = M.glo[mp], hi = M.ghi[mp];
  const double ax = M.gacc[3 * mp], ay = M.gacc[3 * mp + 1], az = M.gacc[3 * mp + 2];
  const int2* o = M.obs + off;
  const int last = n ? o[n - 1].x : -1;
  const int lev = M.klev[g];
  int* cnt = M.counts + (size_t)mp * M.L + lev;
  const int cv = *cnt;
  const double Sl = M.S[lev];
  const long long kf_last = last >= 0 ? M.kf_id[last] : -1;
  if (covis) covis_list(M, slot, o, n, +1, acc);
  // appended after the newest keyframe of a clean (sorted) list: the cached sums extend exactly
  const bool newest = !dirty && (n == 0 || kf_last < kf_new);
  int at = n;
  if (n == cap) {
    const int nc = cap < 4 ? 4 : 2 * cap;
    const int noff = atomicAdd(&M.scal[SC_OBS_HEAD], nc);
    if (noff + nc > M.obs_cap) {
      set_err(M, LM_ERR_CAPACITY);
      return;
    }
    copy_obs(M.obs + noff, o, n);
    M.ooff[mp] = noff;
    M.ocap[mp] = nc;
    M.obs[noff + n] = make_int2(slot, kp);
  } else {
    M.obs[off + at] = make_int2(slot, kp);
  }
  M.nobs[mp] = n + 1;
  M.kbind[g] = mp;
  *cnt = cv + 1;
  M.ver[mp] = vr + 1;
  if (fuse) {
    M.found[mp] = found + 1;
    mark_dirty_owned(M, mp, dirty);
  }
  if (gv && newest) {
    const double rx = px - cx, ry = py - cy, rz = pz - cz;
    const double dd = sqrt(rx * rx + ry * ry + rz * rz);
    if (dd > 0) {  // geo_term
      const double d0 = dd / Sl;
      M.glo[mp] = d0 < lo ? d0 : lo;
      M.ghi[mp] = d0 > hi ? d0 : hi;
      M.gacc[3 * mp] = ax + rx / dd;
      M.gacc[3 * mp + 1] = ay + ry / dd;
      M.gacc[3 * mp + 2] = az + rz / dd;
    }
  } else {
    M.gval[mp] = 0;
  }
}

// fusion's ADD_OBSERVATION (link(fuse=true)) for high-degree points: the lanes share the
// covisibility bumps, lane 0 the record (loads first, as in link). The caller owns mp's
// dirty flag in this phase.
__device__ void link_warp(const DevMap& M, int mp, int slot, int kp, int lane, PairAcc* acc) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  for (int k = lane; k < n; k += 32) covis_add(M, slot, o[k].x, +1, acc);
  __syncwarp();
  if (lane == 0) link(M, mp, slot, kp, acc, true, false);
  __syncwarp();
}

// _unrecord_obs of list entry k: unbind, uncount, covis -1 with every remaining observer
__device__ void unlink_at(const DevMap& M, int mp, int k, PairAcc* acc = nullptr) {
  int2* o = M.obs + M.ooff[mp];
  const int2 e = o[k];
  const int n = M.nobs[mp] - 1;
  for (int m = k; m < n; ++m) o[m] = o[m + 1];
  M.nobs[mp] = n;
  M.gval[mp] = 0;
  M.ver[mp] += 1;
  const int g = M.kp_off[e.x] + e.y;
  M.kbind[g] = -1;
  M.counts[(size_t)mp * M.L + M.klev[g]] -= 1;
  covis_list(M, e.x, o, n, -1, acc);
}

__device__ void kill_point(const DevMap& M, int mp, PairAcc* acc = nullptr) {
  while (M.nobs[mp] > 0) unlink_at(M, mp, 0, acc);
  M.alive[mp] = 0;
}

// replace_map_point(loser, winner); returns migrated observation count
__device__ int replace_point(const DevMap& M, int loser, int winner, PairAcc* acc = nullptr) {
  int migrated = 0;
  while (M.nobs[loser] > 0) {
    const int2 e = M.obs[M.ooff[loser]];
    unlink_at(M, loser, 0, acc);
    if (obs_find(M, winner, e.x) >= 0) continue;  // winner sees this keyframe: slot stays unbound
    link(M, winner, e.x, e.y, acc);
    ++migrated;
  }
  M.found[winner] += M.found[loser];
  M.visible[winner] += M.visible[loser];
  M.alive[loser] = 0;
  M.mrg[loser] = make_int2(M.scal[SC_MTAG], winner);
  mark_dirty(M, winner);
  return migrated;
}

// fusion._merge: more observations wins, ties lose the higher id; winner found += 1
__device__ void merge_pair(const DevMap& M, int a, int b, PairAcc* acc = nullptr) {
  const int na = M.nobs[a], nb = M.nobs[b];
  int loser, winner;
  if (na == nb) {
    loser = a > b ? a : b;
    winner = a > b ? b : a;
  } else if (na < nb) {
    loser = a;
    winner = b;
  } else {
    loser = b;
    winner = a;
  }
  replace_point(M, loser, winner, acc);
  M.found[winner] += 1;
}

// ------------------------------------------------------------ warp-cooperative kill / merge
// Same net effect as the sequential unlink/link loops above (all covisibility bumps are
// commutative), with the O(n^2) pair work spread over the 32 lanes of one warp.

// covisibility delta d for every unordered pair of o[0..n) (warp; n <= 64 from registers:
// lane l holds entries l and l+32, entry a is broadcast by a shuffle)
__device__ void covis_pairs_warp(const DevMap& M, const int2* o, int n, int d, int lane, PairAcc* acc) {
  if (n <= 64) {
    const int s0 = lane < n ? o[lane].x : -1, s1 = lane + 32 < n ? o[lane + 32].x : -1;
    for (int a = 0; a < n - 1; ++a) {
      const int sa = __shfl_sync(0xffffffffu, a < 32 ? s0 : s1, a & 31);
      if (lane > a && lane < n) covis_add(M, sa, s0, d, acc);
      if (lane + 32 > a && lane + 32 < n) covis_add(M, sa, s1, d, acc);
    }
    return;
  }
  for (int a = 0; a < n; ++a)
    for (int b = a + 1 + lane; b < n; b += 32) covis_add(M, o[a].x, o[b].x, d, acc);
}

// covisibility delta d for every pair (x in oa[0..na), y in ob[0..nb)) (warp; nb <= 64 from
// registers, oa entries broadcast one by one)
__device__ void covis_cross_warp(const DevMap& M, const int2* oa, int na, const int2* ob, int nb, int d, int lane,
                                 PairAcc* acc) {
  if (nb <= 64) {
    const int t0 = lane < nb ? ob[lane].x : -1, t1 = lane + 32 < nb ? ob[lane + 32].x : -1;
    for (int a0 = 0; a0 < na; a0 += 32) {
      const int sv = a0 + lane < na ? oa[a0 + lane].x : -1;
      const int m = na - a0 < 32 ? na - a0 : 32;
      for (int a = 0; a < m; ++a) {
        const int sa = __shfl_sync(0xffffffffu, sv, a);
        if (lane < nb) covis_add(M, sa, t0, d, acc);
        if (lane + 32 < nb) covis_add(M, sa, t1, d, acc);
      }
    }
    return;
  }
  for (int q = lane; q < na * nb; q += 32) covis_add(M, oa[q / nb].x, ob[q % nb].x, d, acc);
}

// kill_map_point (mapmodel.py:233-237) of a point with at most KT observations, one thread
template <int KT>
__device__ void kill_point_thread(const DevMap& M, int mp, PairAcc* acc) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  int sl[KT], kp[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k)
    if (k < n) {
      const int2 e = o[k];
      sl[k] = e.x;
      kp[k] = e.y;
    }
#pragma unroll
  for (int a = 0; a < KT; ++a)
#pragma unroll
    for (int b = a + 1; b < KT; ++b)
      if (b < n) covis_add(M, sl[a], sl[b], -1, acc);
#pragma unroll
  for (int k = 0; k < KT; ++k)
    if (k < n) M.kbind[M.kp_off[sl[k]] + kp[k]] = -1;
  for (int l = 0; l < M.L; ++l) M.counts[(size_t)mp * M.L + l] = 0;
  M.nobs[mp] = 0;
  M.alive[mp] = 0;
  M.gval[mp] = 0;
  M.ver[mp] += 1;
}

// kill_map_point without its covisibility update, for a batch of kills whose observers all
// lie in the accumulator's window: the point's observer set goes to row[0..2] (96-bit mask
// over window slots) and the caller subtracts the pair counts of all rows at once (a Gram
// matrix of the masks). Returns false (nothing done) when an observer is outside the window.
__device__ bool kill_point_rows_warp(const DevMap& M, int mp, int lane, const PairAcc* acc, unsigned* row) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  unsigned r[3] = {0u, 0u, 0u};
  bool inside = true;
  for (int k = lane; k < n; k += 32) {
    const int w = o[k].x - acc->wbase;
    inside &= w >= 0 && w < PAIR_W;
    if (w >= 0 && w < PAIR_W) r[w >> 5] |= 1u << (w & 31);
  }
  if (!__all_sync(0xffffffffu, inside)) return false;
#pragma unroll
  for (int q = 0; q < 3; ++q) r[q] = __reduce_or_sync(0xffffffffu, r[q]);
  for (int k = lane; k < n; k += 32) M.kbind[M.kp_off[o[k].x] + o[k].y] = -1;
  for (int l = lane; l < M.L; l += 32) M.counts[(size_t)mp * M.L + l] = 0;
  __syncwarp();
  if (lane == 0) {
    row[0] = r[0];
    row[1] = r[1];
    row[2] = r[2];
    M.nobs[mp] = 0;
    M.alive[mp] = 0;
    M.gval[mp] = 0;
    M.ver[mp] += 1;
  }
  __syncwarp();
  return true;
}

// the same, one thread (entries loaded 8 at a time)
__device__ bool kill_point_rows_thread(const DevMap& M, int mp, const PairAcc* acc, unsigned* row) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  unsigned r0 = 0u, r1 = 0u, r2 = 0u;
  for (int k0 = 0; k0 < n; k0 += 8) {
    int2 e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = k0 + j < n ? o[k0 + j] : make_int2(acc->wbase, 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (k0 + j >= n) continue;
      const int w = e[j].x - acc->wbase;
      if (w < 0 || w >= PAIR_W) return false;
      r0 |= w < 32 ? 1u << w : 0u;
      r1 |= w >= 32 && w < 64 ? 1u << (w - 32) : 0u;
      r2 |= w >= 64 ? 1u << (w - 64) : 0u;
    }
  }
  for (int k0 = 0; k0 < n; k0 += 8) {
    int2 e[8];
    int g[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = k0 + j < n ? o[k0 + j] : make_int2(0, 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = k0 + j < n ? M.kp_off[e[j].x] + e[j].y : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (k0 + j < n) M.kbind[g[j]] = -1;
  }
  for (int l = 0; l < M.L; ++l) M.counts[(size_t)mp * M.L + l] = 0;
  row[0] = r0;
  row[1] = r1;
  row[2] = r2;
  M.nobs[mp] = 0;
  M.alive[mp] = 0;
  M.gval[mp] = 0;
  M.ver[mp] += 1;
  return true;
}

// kill_map_point (mapmodel.py:233-237), all lanes of a warp call it with the same mp
__device__ void kill_point_warp(const DevMap& M, int mp, int lane, PairAcc* acc) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  covis_pairs_warp(M, o, n, -1, lane, acc);
  for (int k = lane; k < n; k += 32) M.kbind[M.kp_off[o[k].x] + o[k].y] = -1;
  for (int l = lane; l < M.L; l += 32) M.counts[(size_t)mp * M.L + l] = 0;
  __syncwarp();
  if (lane == 0) {
    M.nobs[mp] = 0;
    M.alive[mp] = 0;
    M.gval[mp] = 0;
    M.ver[mp] += 1;
  }
  __syncwarp();
}

// fusion._merge (fusion.py) = replace_map_point(loser, winner) (mapmodel.py:245-267) + the
// winner's found bump, warp-cooperative. Every scalar of both points is loaded in one first
// round (the stores below would otherwise serialise the loads); the caller owns both points
// in this phase (exclusive reservations), so the winner's dirty flag is set without an atomic
// exchange.
__device__ void merge_pair_warp(const DevMap& M, int a, int b, int lane, PairAcc* acc) {
  const int na = M.nobs[a], nb = M.nobs[b], fa = M.ooff[a], fb = M.ooff[b], ca = M.ocap[a], cb = M.ocap[b];
  const int ua = M.found[a], ub = M.found[b], va = M.visible[a], vb = M.visible[b];
  const int ra = M.ver[a], rb = M.ver[b], da = M.dirty[a], db = M.dirty[b];
  const int mtag = M.scal[SC_MTAG];
  const bool la = na == nb ? a > b : na < nb;  // a loses (fewer observations; tie: larger id)
  const int loser = la ? a : b, winner = la ? b : a;
  const int nL = la ? na : nb, nW = la ? nb : na, offW = la ? fb : fa, capW = la ? cb : ca;
  int2* oL = M.obs + (la ? fa : fb);
  const int2* oW = M.obs + offW;
  // (a) covisibility -1 for every pair of the loser's observers
  covis_pairs_warp(M, oL, nL, -1, lane, acc);
  __syncwarp();
  // (b) migrate the observations of keyframes the winner does not see; compact them in place
  int nM = 0;
  for (int c0 = 0; c0 < nL; c0 += 32) {
    const int k = c0 + lane;
    int2 e = make_int2(0, 0);
    bool mig = false;
    if (k < nL) {
      e = oL[k];
      mig = true;
      for (int w0 = 0; w0 < nW; w0 += 8) {  // winner entries 8 at a time (broadcast loads)
        int sw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) sw[j] = w0 + j < nW ? oW[w0 + j].x : -1;
#pragma unroll
        for (int j = 0; j < 8; ++j) mig &= sw[j] != e.x;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, mig);
    __syncwarp();
    if (k < nL) {
      const int g = M.kp_off[e.x] + e.y;
      M.kbind[g] = mig ? winner : -1;
      if (mig) {
        atomicAdd(&M.counts[(size_t)winner * M.L + M.klev[g]], 1);
        oL[nM + __popc(bal & ((1u << lane) - 1))] = e;
      }
    }
    nM += __popc(bal);
    __syncwarp();
  }
  // (c) covisibility +1: migrated x winner's original observers, and migrated pairs
  covis_cross_warp(M, oL, nM, oW, nW, +1, lane, acc);
  covis_pairs_warp(M, oL, nM, +1, lane, acc);
  // (d) winner list += migrated observations (appended; the winner is marked dirty, so the
  //     list is re-sorted by keyframe id before any order-dependent read)
  int nWn = nW, offWn = offW, capWn = capW;
  if (nM > 0) {
    int off = offW, cap = capW;
    if (lane == 0 && nW + nM > capW) {
      int nc = capW < 4 ? 4 : capW;
      while (nc < nW + nM) nc *= 2;
      off = atomicAdd(&M.scal[SC_OBS_HEAD], nc);
      if (off + nc > M.obs_cap) {
        set_err(M, LM_ERR_CAPACITY);
        off = -1;
      }
      cap = nc;
    }
    off = __shfl_sync(0xffffffffu, off, 0);
    cap = __shfl_sync(0xffffffffu, cap, 0);
    if (off >= 0) {
      int2* B = M.obs + off;
      if (off != offW)
        for (int i = lane; i < nW; i += 32) B[i] = oW[i];
      for (int j = lane; j < nM; j += 32) B[nW + j] = oL[j];
      nWn = nW + nM;
      offWn = off;
      capWn = cap;
    }
  }
  __syncwarp();
  for (int l = lane; l < M.L; l += 32) M.counts[(size_t)loser * M.L + l] = 0;
  if (lane == 0) {
    M.ooff[winner] = offWn;
    M.ocap[winner] = capWn;
    M.nobs[winner] = nWn;
    M.nobs[loser] = 0;
    M.found[winner] = ua + ub + 1;  // found(winner) + found(loser), then _merge's own bump
    M.visible[winner] = va + vb;
    M.alive[loser] = 0;
    M.mrg[loser] = make_int2(mtag, winner);
    M.gval[winner] = 0;
    M.gval[loser] = 0;
    M.ver[winner] = (la ? rb : ra) + 1;
    M.ver[loser] = (la ? ra : rb) + 1;
    mark_dirty_owned(M, winner, la ? db : da);
  }
  __syncwarp();
}

// k-th smallest of d[0..n) (quickselect, d is scratch)
__device__ int kth_smallest(unsigned short* d, int n, int k) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const unsigned short pivot = d[(lo + hi) >> 1];
    int i = lo, j = hi;
    while (i <= j) {
      while (d[i] < pivot) ++i;
      while (d[j] > pivot) --j;
      if (i <= j) {
        const unsigned short tmp = d[i];
        d[i] = d[j];
        d[j] = tmp;
        ++i;
        --j;
      }
    }
    if (k <= j)
      hi = j;
    else if (k >= i)
      lo = i;
    else
      return d[k];
  }
  return d[k];
}

// sort the observation list of mp by keyframe id (warp-cooperative rank scatter; ids are
// distinct). Lists longer than 128 fall back to an insertion sort on lane 0.
__device__ void sort_obs_warp(const DevMap& M, int2* o, int n, int lane) {
  if (n <= 1) return;
  if (n > 128) {
    if (lane == 0)
      for (int i = 1; i < n; ++i) {
        const int2 e = o[i];
        const long long ke = M.kf_id[e.x];
        int k = i;
        while (k > 0 && M.kf_id[o[k - 1].x] > ke) {
          o[k] = o[k - 1];
          --k;
        }
        o[k] = e;
      }
    __syncwarp();
    return;
  }
  int2 e[4];
  int r[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = lane + 32 * c;
    r[c] = -1;
    if (i < n) {
      e[c] = o[i];
      const long long ki = M.kf_id[e[c].x];
      int rk = 0;
      for (int j = 0; j < n; ++j) rk += M.kf_id[o[j].x] < ki;
      r[c] = rk;
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (r[c] >= 0) o[r[c]] = e[c];
  __syncwarp();
}

// warp-parallel geometry-cache rebuild (sorted list): lanes compute the per-observation
// terms, lane 0 accumulates them in list order (the reference's order) -> bit-identical
__device__ void geo_full_warp(const DevMap& M, int mp, int lane) {
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  double lo = INFINITY, hi = -INFINITY, ax = 0, ay = 0, az = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int k = c0 + lane;
    double rx = 0, ry = 0, rz = 0, dd = 1, d0 = 0;
    bool ok = false;
    if (k < n) ok = geo_term(M, mp, o[k], rx, ry, rz, dd, d0);
    const double tx = ok ? rx / dd : 0, ty = ok ? ry / dd : 0, tz = ok ? rz / dd : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const int cn = n - c0 < 32 ? n - c0 : 32;
    for (int q = 0; q < cn; ++q) {
      const double sx = __shfl_sync(0xffffffffu, tx, q), sy = __shfl_sync(0xffffffffu, ty, q);
      const double sz = __shfl_sync(0xffffffffu, tz, q), s0 = __shfl_sync(0xffffffffu, d0, q);
      if (bal >> q & 1u) {
        lo = s0 < lo ? s0 : lo;
        hi = s0 > hi ? s0 : hi;
        ax = ax + sx;
        ay = ay + sy;
        az = az + sz;
      }
    }
  }
  if (lane == 0) {
    M.gacc[3 * mp] = ax;
    M.gacc[3 * mp + 1] = ay;
    M.gacc[3 * mp + 2] = az;
    M.glo[mp] = lo;
    M.ghi[mp] = hi;
    M.gval[mp] = 1;
  }
  __syncwarp();
}

// _refresh_rep_descriptor, one warp per point: the observing descriptor whose median
// Hamming distance to the others is smallest (first in (kf id) order wins). The median of
// the n-1 integer distances is compared as the sum of the two middle order statistics,
// which orders exactly like the reference's float nanmedian. Sorts the list first.
// k-th smallest (k from 0) of the 9-bit values whose bit-planes are pl[bit][word] over the
// candidate set cand[word]: radix select, 9 steps of popcounts (registers only)
template <int NW>
__device__ __forceinline__ int plane_select(const unsigned (&pl)[9][NW], unsigned (&cand)[NW], int k) {
  int v = 0;
#pragma unroll
  for (int bit = 8; bit >= 0; --bit) {
    int c0 = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) c0 += __popc(cand[w] & ~pl[bit][w]);
    const bool zero = k < c0;
    if (!zero) {
      k -= c0;
      v |= 1 << bit;
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) cand[w] &= zero ? ~pl[bit][w] : pl[bit][w];
  }
  return v;
}

// Representative descriptor, all in registers (3 <= n <= 32*NW): d(a, b) = d(b, a), so every unordered pair is
// popcounted once. Row slot s of lane l is observation 32*s + l. Diagonal blocks (s, s):
// in step r (1..16) lane l computes d(l, l+r mod 32) for its own row and hands it to lane
// l+r (shuffle) for that lane's row; off-diagonal blocks (s1 < s2): in step r (0..31) lane l
// computes d(32*s1 + l, 32*s2 + (l+r mod 32)) and hands it to lane l+r's row slot s2. Half the
// popcounts of the row-by-row version (the pipe that bounds it, 16 lanes/clk/SM).
template <int NW>
__device__ void refresh_rep_sym(const DevMap& M, int2* o, int n, uint4* rep, int lane) {
  int2 e[NW];
  long long key[NW];
  uint4 d0[NW], d1[NW];
#pragma unroll
  for (int s = 0; s < NW; ++s) e[s] = s * 32 + lane < n ? o[s * 32 + lane] : make_int2(0, 0);
#pragma unroll
  for (int s = 0; s < NW; ++s) {
    const bool act = s * 32 + lane < n;
    key[s] = act ? M.kf_id[e[s].x] : 0x7fffffffffffffffll;
    const int g = M.kp_off[e[s].x] + e[s].y;
    d0[s] = act ? M.kdesc[2 * g] : make_uint4(0, 0, 0, 0);
    d1[s] = act ? M.kdesc[2 * g + 1] : make_uint4(0, 0, 0, 0);
  }
  int rk[NW];
#pragma unroll
  for (int s = 0; s < NW; ++s) rk[s] = 0;
#pragma unroll
  for (int sb = 0; sb < NW; ++sb)
#pragma unroll 4
    for (int l = 0; l < 32; ++l) {
      const long long kb = __shfl_sync(0xffffffffu, key[sb], l);
#pragma unroll
      for (int s = 0; s < NW; ++s) rk[s] += kb < key[s];
    }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < NW; ++s)
    if (s * 32 + lane < n) o[rk[s]] = e[s];
  unsigned pl[NW][9][NW];  // [row slot][bit][column word]
#pragma unroll
  for (int s = 0; s < NW; ++s)
#pragma unroll
    for (int bit = 0; bit < 9; ++bit)
#pragma unroll
      for (int w = 0; w < NW; ++w) pl[s][bit][w] = 0u;
#pragma unroll
  for (int s1 = 0; s1 < NW; ++s1)
#pragma unroll
    for (int s2 = s1; s2 < NW; ++s2) {
      const int r0 = s1 == s2 ? 1 : 0, r1 = s1 == s2 ? 16 : 31;
#pragma unroll 2
      for (int r = r0; r <= r1; ++r) {
        const int src = (lane + r) & 31, from = (lane - r) & 31;
        uint4 b0, b1;
        b0.x = __shfl_sync(0xffffffffu, d0[s2].x, src);
        b0.y = __shfl_sync(0xffffffffu, d0[s2].y, src);
        b0.z = __shfl_sync(0xffffffffu, d0[s2].z, src);
        b0.w = __shfl_sync(0xffffffffu, d0[s2].w, src);
        b1.x = __shfl_sync(0xffffffffu, d1[s2].x, src);
        b1.y = __shfl_sync(0xffffffffu, d1[s2].y, src);
        b1.z = __shfl_sync(0xffffffffu, d1[s2].z, src);
        b1.w = __shfl_sync(0xffffffffu, d1[s2].w, src);
        const unsigned dist = (unsigned)hamming(d0[s1], d1[s1], b0, b1);  // d(32*s1+lane, 32*s2+src)
        const unsigned got = __shfl_sync(0xffffffffu, dist, from);       // d(32*s1+from, 32*s2+lane)
#pragma unroll
        for (int bit = 0; bit < 9; ++bit) {
          pl[s1][bit][s2] |= ((dist >> bit) & 1u) << src;
          if (!(s1 == s2 && r == 16)) pl[s2][bit][s1] |= ((got >> bit) & 1u) << from;
        }
      }
    }
  const int m = n - 1, k0 = (m - 1) >> 1, k1 = m >> 1;
  unsigned best = 0xffffffffu;
#pragma unroll
  for (int s = 0; s < NW; ++s) {
    const int i = s * 32 + lane;
    if (i < n) {
      unsigned cand[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {  // the other real observations
        const int lo = w * 32;
        unsigned msk = n - lo >= 32 ? 0xffffffffu : (n - lo <= 0 ? 0u : (1u << (n - lo)) - 1u);
        if (i >= lo && i < lo + 32) msk &= ~(1u << (i - lo));
        cand[w] = msk;
      }
      unsigned c2[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) c2[w] = cand[w];
      const int v0 = plane_select<NW>(pl[s], cand, k0);
      const int v1 = k1 == k0 ? v0 : plane_select<NW>(pl[s], c2, k1);
      const unsigned kk = ((unsigned)(v0 + v1) << 16) | (unsigned)rk[s];
      best = kk < best ? kk : best;
    }
  }
  for (int off = 16; off; off >>= 1) {
    const unsigned other = __shfl_xor_sync(0xffffffffu, best, off);
    best = other < best ? other : best;
  }
#pragma unroll
  for (int s = 0; s < NW; ++s)
    if (s * 32 + lane < n && rk[s] == (int)(best & 0xffffu)) {
      rep[0] = d0[s];
      rep[1] = d1[s];
    }
  __syncwarp();
}

// refresh for 32 < n <= 32*NS observations: lane l holds observations l, l+32, ...
// (entry, key, descriptor in registers); every row's distances come from broadcast
// descriptors (no dependent global loads), its two middle order statistics from a
// quickselect over a per-lane scratch row (L1-resident local memory).
template <int NS>
__device__ void refresh_rep_lanes(const DevMap& M, int2* o, int n, uint4* rep, int lane) {
  int2 e[NS];
  long long key[NS];
  uint4 d0[NS], d1[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int i = s * 32 + lane;
    e[s] = i < n ? o[i] : make_int2(0, 0);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int i = s * 32 + lane;
    key[s] = i < n ? M.kf_id[e[s].x] : 0x7fffffffffffffffll;
    const int g = M.kp_off[e[s].x] + e[s].y;
    d0[s] = i < n ? M.kdesc[2 * g] : make_uint4(0, 0, 0, 0);
    d1[s] = i < n ? M.kdesc[2 * g + 1] : make_uint4(0, 0, 0, 0);
  }
  int rk[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) rk[s] = 0;
#pragma unroll
  for (int sb = 0; sb < NS; ++sb)
    for (int l = 0; l < 32; ++l) {
      const long long kb = __shfl_sync(0xffffffffu, key[sb], l);
#pragma unroll
      for (int s = 0; s < NS; ++s) rk[s] += kb < key[s];
    }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s * 32 + lane < n) o[rk[s]] = e[s];
  unsigned short d[NS][32 * NS];
#pragma unroll
  for (int sb = 0; sb < NS; ++sb)
    for (int l = 0; l < 32; ++l) {
      uint4 b0, b1;
      b0.x = __shfl_sync(0xffffffffu, d0[sb].x, l);
      b0.y = __shfl_sync(0xffffffffu, d0[sb].y, l);
      b0.z = __shfl_sync(0xffffffffu, d0[sb].z, l);
      b0.w = __shfl_sync(0xffffffffu, d0[sb].w, l);
      b1.x = __shfl_sync(0xffffffffu, d1[sb].x, l);
      b1.y = __shfl_sync(0xffffffffu, d1[sb].y, l);
      b1.z = __shfl_sync(0xffffffffu, d1[sb].z, l);
      b1.w = __shfl_sync(0xffffffffu, d1[sb].w, l);
      const int b = sb * 32 + l;
#pragma unroll
      for (int s = 0; s < NS; ++s) d[s][b] = (unsigned short)hamming(d0[s], d1[s], b0, b1);
    }
  const int m = n - 1, k0 = (m - 1) >> 1, k1 = m >> 1;
  unsigned best = 0xffffffffu;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int i = s * 32 + lane;
    if (i >= n) continue;
    unsigned short* r = d[s];
    r[i] = r[n - 1];  // drop the self distance: the last real entry moves into its place
    const int v0 = kth_smallest(r, m, k0);
    int v1 = v0;
    if (k1 != k0) {
      v1 = 0x7fffffff;
      for (int b = k0 + 1; b < m; ++b) v1 = r[b] < v1 ? r[b] : v1;
    }
    const unsigned kk = ((unsigned)(v0 + v1) << 16) | (unsigned)rk[s];
    best = kk < best ? kk : best;
  }
  for (int off = 16; off; off >>= 1) {
    const unsigned other = __shfl_xor_sync(0xffffffffu, best, off);
    best = other < best ? other : best;
  }
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s * 32 + lane < n && rk[s] == (int)(best & 0xffffu)) {
      rep[0] = d0[s];
      rep[1] = d1[s];
    }
  __syncwarp();
}

// refresh_rep_list for lists longer than REFRESH_MAXN (no per-row distance array): each
// row's two middle order statistics by a 9-bit radix select whose every step recounts the
// row's distances (recomputed popcounts), so memory stays O(1) per lane for any n. Slow
// (~11 passes over the list per row) but exact; only points observed by > 512 keyframes
// take it. o must already be sorted by keyframe id.
__device__ void refresh_rep_radix(const DevMap& M, const int2* o, int n, uint4* rep, int lane) {
  const int m = n - 1, k0 = (m - 1) >> 1, k1 = m >> 1;
  unsigned best = 0xffffffffu;  // (med2 << 16) | row
  for (int a = lane; a < n; a += 32) {
    const int ga = M.kp_off[o[a].x] + o[a].y;
    const uint4 a0 = M.kdesc[2 * ga], a1 = M.kdesc[2 * ga + 1];
    auto dist = [&](int b) -> int {
      const int gb = M.kp_off[o[b].x] + o[b].y;
      return hamming(a0, a1, M.kdesc[2 * gb], M.kdesc[2 * gb + 1]);
    };
    // k0-th smallest (from 0) of d(a, b), b != a
    int prefix = 0, k = k0;
    for (int bit = 8; bit >= 0; --bit) {
      int c0 = 0;
      for (int b = 0; b < n; ++b) {
        if (b == a) continue;
        const int d = dist(b);
        c0 += (d >> (bit + 1)) == prefix && !((d >> bit) & 1);
      }
      if (k < c0) {
        prefix = prefix << 1;
      } else {
        k -= c0;
        prefix = (prefix << 1) | 1;
      }
    }
    const int v0 = prefix;
    int v1 = v0;
    if (k1 != k0) {  // next order statistic: v0 again if it repeats, else the smallest larger value
      int le = 0, nxt = 0x7fffffff;
      for (int b = 0; b < n; ++b) {
        if (b == a) continue;
        const int d = dist(b);
        le += d <= v0;
        if (d > v0 && d < nxt) nxt = d;
      }
      v1 = le > k1 ? v0 : nxt;
    }
    const unsigned key = ((unsigned)(v0 + v1) << 16) | (unsigned)a;
    best = key < best ? key : best;
  }
  for (int off = 16; off; off >>= 1) {
    const unsigned other = __shfl_xor_sync(0xffffffffu, best, off);
    best = other < best ? other : best;
  }
  if (lane == 0) {
    const int a = best & 0xffff;
    const int g = M.kp_off[o[a].x] + o[a].y;
    rep[0] = M.kdesc[2 * g];
    rep[1] = M.kdesc[2 * g + 1];
  }
  __syncwarp();
}

// _refresh_rep_descriptor of the observation list o[0..n) (sorted in place by keyframe id),
// result into rep[0..1]; one warp
__device__ void refresh_rep_list(const DevMap& M, int2* o, int n, uint4* rep, int lane) {
  if (n >= 3 && n <= 32) return refresh_rep_sym<1>(M, o, n, rep, lane);
  if (n >= 33 && n <= 64) return refresh_rep_sym<2>(M, o, n, rep, lane);
  if (n >= 65 && n <= 128) return refresh_rep_lanes<4>(M, o, n, rep, lane);
  sort_obs_warp(M, o, n, lane);
  if (n == 0) return;
  if (n <= 2) {  // one observation, or two (equal medians -> the first)
    if (lane == 0) {
      const int g = M.kp_off[o[0].x] + o[0].y;
      rep[0] = M.kdesc[2 * g];
      rep[1] = M.kdesc[2 * g + 1];
    }
    __syncwarp();
    return;
  }
  if (n > REFRESH_MAXN) return refresh_rep_radix(M, o, n, rep, lane);
  unsigned short d[REFRESH_MAXN];
  const int m = n - 1, k0 = (m - 1) >> 1, k1 = m >> 1;
  unsigned best = 0xffffffffu;  // (med2 << 16) | row
  for (int a = lane; a < n; a += 32) {
    const int ga = M.kp_off[o[a].x] + o[a].y;
    const uint4 a0 = M.kdesc[2 * ga], a1 = M.kdesc[2 * ga + 1];
    int c = 0;
    for (int b = 0; b < n; ++b) {
      if (b == a) continue;
      const int gb = M.kp_off[o[b].x] + o[b].y;
      d[c++] = (unsigned short)hamming(a0, a1, M.kdesc[2 * gb], M.kdesc[2 * gb + 1]);
    }
    const int v0 = kth_smallest(d, m, k0);
    int v1 = v0;
    if (k1 != k0) {  // next order statistic: min of the upper partition
      v1 = 0x7fffffff;
      for (int b = k0 + 1; b < m; ++b) v1 = d[b] < v1 ? d[b] : v1;
    }
    const unsigned key = ((unsigned)(v0 + v1) << 16) | (unsigned)a;
    best = key < best ? key : best;
  }
  for (int off = 16; off; off >>= 1) {
    const unsigned other = __shfl_xor_sync(0xffffffffu, best, off);
    best = other < best ? other : best;
  }
  if (lane == 0) {
    const int a = best & 0xffff;
    const int g = M.kp_off[o[a].x] + o[a].y;
    rep[0] = M.kdesc[2 * g];
    rep[1] = M.kdesc[2 * g + 1];
  }
  __syncwarp();
}

__device__ void refresh_rep_warp(const DevMap& M, int mp, int lane) {
  refresh_rep_list(M, M.obs + M.ooff[mp], M.nobs[mp], M.rep + 2 * (size_t)mp, lane);
}

}  // namespace lm
