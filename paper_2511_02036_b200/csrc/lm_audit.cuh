// lm_audit.cuh -- device-side MapModel.audit (pkg/src/localmap/mapmodel.py:304-353).
//
// The reference rechecks, by brute force over its Python dicts, that the map's redundant
// bookkeeping agrees with itself. The device map holds the same redundancy (observation
// lists, slot bindings, per-level counters, dense covisibility), so the same checks run as
// three wide kernels over the device state, appending violation records {code, a, b, c}
// that the host formats with the reference's messages:
//   k_audit_points  thread per map point: a dead point keeps no observations; every
//                   observation of a live point is in a live keyframe whose slot binds the
//                   point; the per-level counter row equals the histogram of its observations'
//                   levels (and sums to their number); covisibility pairs of its bound
//                   observers counted into an expected matrix E
//   k_audit_slots   thread per keypoint of a live keyframe: a bound slot names a live point
//                   that lists (keyframe, slot) among its observations
//   k_audit_covis   thread per live keyframe pair: covis[a][b] == E[a][b] (= the number of
//                   live points bound in both, the reference's set intersection)
#pragma once
#include "lm_map.cuh"

namespace lm {

enum AuditCode {
  AV_DEAD_OBS = 1,       // dead map point {mp} retains observations
  AV_OBS_DEAD_KF = 2,    // map point {mp} observes dead keyframe {slot}
  AV_BIND_MISMATCH = 3,  // binding mismatch: map point {mp} vs slot ({slot}, {kp})
  AV_COUNTS = 4,         // scale_counts mismatch for map point {mp}
  AV_COUNTS_SUM = 5,     // scale_counts sum mismatch for map point {mp}
  AV_SLOT_DEAD = 6,      // slot ({slot}, {kp}) bound to dead point {mp}
  AV_SLOT_NOT_OBS = 7,   // slot ({slot}, {kp}) not in map point {mp} observations
  AV_COVIS = 8           // covisibility weight mismatch for pair ({slot a}, {slot b})
};

struct AuditOut {
  int* count;  // [1] violations found (may exceed cap)
  int4* rec;   // [cap]
  int cap;
  int* expect; // [kf_cap * kf_cap] expected covisibility (upper triangle used)
};

__device__ __forceinline__ void audit_emit(const AuditOut& O, int code, int a, int b, int c) {
  const int at = atomicAdd(O.count, 1);
  if (at < O.cap) O.rec[at] = make_int4(code, a, b, c);
}

__global__ void __launch_bounds__(256) k_audit_points(DevMap M, AuditOut O, int n_points) {
  const int mp = blockIdx.x * 256 + threadIdx.x;
  if (mp >= n_points) return;
  const int2* o = M.obs + M.ooff[mp];
  const int n = M.nobs[mp];
  if (!M.alive[mp]) {
    if (n) audit_emit(O, AV_DEAD_OBS, mp, 0, 0);
    return;
  }
  int expect[LMAX];
  for (int l = 0; l < LMAX; ++l) expect[l] = 0;
  for (int k = 0; k < n; ++k) {
    const int slot = o[k].x, kp = o[k].y;
    if (M.kf_state[slot] != KF_LIVE) {
      audit_emit(O, AV_OBS_DEAD_KF, mp, slot, 0);
      continue;
    }
    const int g = M.kp_off[slot] + kp;
    if (M.kbind[g] != mp) audit_emit(O, AV_BIND_MISMATCH, mp, slot, kp);
    expect[M.klev[g]] += 1;
  }
  int sum = 0;
  bool eq = true;
  for (int l = 0; l < M.L; ++l) {
    const int c = M.counts[(size_t)mp * M.L + l];
    eq &= c == expect[l];
    sum += c;
  }
  if (!eq) audit_emit(O, AV_COUNTS, mp, 0, 0);
  if (sum != n) audit_emit(O, AV_COUNTS_SUM, mp, 0, 0);
  // expected covisibility: every pair of live keyframes whose slot binds this point
  for (int a = 0; a < n; ++a) {
    const int sa = o[a].x;
    if (M.kf_state[sa] != KF_LIVE || M.kbind[M.kp_off[sa] + o[a].y] != mp) continue;
    for (int b = a + 1; b < n; ++b) {
      const int sb = o[b].x;
      if (sb == sa || M.kf_state[sb] != KF_LIVE || M.kbind[M.kp_off[sb] + o[b].y] != mp) continue;
      const int lo = sa < sb ? sa : sb, hi = sa < sb ? sb : sa;
      atomicAdd(&O.expect[(size_t)lo * M.kf_cap + hi], 1);
    }
  }
}

// grid-stride over the keypoints of the live keyframes (slot-major)
__global__ void __launch_bounds__(256) k_audit_slots(DevMap M, AuditOut O, int n_slots, int n_points) {
  for (int slot = blockIdx.y; slot < n_slots; slot += gridDim.y) {
    if (M.kf_state[slot] != KF_LIVE) continue;
    const int off = M.kp_off[slot], n = M.kp_n[slot];
    for (int kp = blockIdx.x * 256 + threadIdx.x; kp < n; kp += gridDim.x * 256) {
      const int mp = M.kbind[off + kp];
      if (mp < 0) continue;
      if (mp >= n_points || !M.alive[mp]) {
        audit_emit(O, AV_SLOT_DEAD, slot, kp, mp);
        continue;
      }
      const int2* o = M.obs + M.ooff[mp];
      const int no = M.nobs[mp];
      int at = -1;
      for (int k = 0; k < no; ++k)
        if (o[k].x == slot) at = o[k].y;
      if (at != kp) audit_emit(O, AV_SLOT_NOT_OBS, slot, kp, mp);
    }
  }
}

__global__ void __launch_bounds__(256) k_audit_covis(DevMap M, AuditOut O, int n_slots) {
  const long long np = (long long)n_slots * n_slots;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < np; e += (long long)gridDim.x * 256) {
    const int a = (int)(e / n_slots), b = (int)(e - (long long)a * n_slots);
    if (b <= a || M.kf_state[a] != KF_LIVE || M.kf_state[b] != KF_LIVE) continue;
    const int want = O.expect[(size_t)a * M.kf_cap + b];
    if (M.covis[(size_t)a * M.kf_cap + b] != want || M.covis[(size_t)b * M.kf_cap + a] != want)
      audit_emit(O, AV_COVIS, a, b, 0);
  }
}

}  // namespace lm
