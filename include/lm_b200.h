/* lm_b200.h -- C ABI of the B200-native local-mapping hot path (CreateNewMapPoints +
 * SearchAndFuse of arXiv 2511.02036, reference package `localmap`).
 *
 * A context owns one CUDA device, one stream and a set of device-resident maps
 * ("sessions"). Each map is a structure-of-arrays store of keyframes (poses, pinhole
 * intrinsics, keypoints, 256-bit descriptors, per-keyframe cell grids), map points
 * (positions, representative descriptors, observation lists, per-level counters) and a
 * dense covisibility matrix. All buffers are allocated once at map creation.
 *
 * Conventions: plain C types, explicit sizes, no exceptions. Every function returns an
 * lm_status; on failure lm_last_error(ctx) holds a message. Map point ids and keyframe
 * ids are int64 like the reference's Python ints. Descriptors are 32 bytes per keypoint.
 *
 * Reference entry points each call replaces (paths under pkg/src/localmap/):
 *   lm_kf_stage + lm_kf_insert   MapModel.insert_keyframe mapmodel.py:185-199 and
 *                                DeviceStore.upload_keyframe devicestore.py:68-78
 *   lm_create_map_points         create_map_points triangulation.py:195-300
 *   lm_search                    search_for_triangulation triangulation.py:80-114
 *   lm_run_fusion                run_fusion fusion.py:307-347
 *   lm_fusion_targets            collect_fusion_targets fusion.py:38-54
 *   lm_fuse_pass                 fuse_pass fusion.py:132-175
 *   lm_apply_fusion              apply_fusion fusion.py:249-292
 *   lm_cull_recent               cull_recent_map_points culling.py:28-59
 *   lm_step / lm_step_batch      one pipeline iteration pipeline.py:152-195 (insert, recent
 *                                cull, triangulation, fusion; LBA and keyframe culling are
 *                                out of scope)
 *   lm_mp_new / lm_obs_add / lm_obs_erase / lm_mp_kill / lm_mp_replace
 *                                MapModel ops mapmodel.py:201-267
 *   lm_covisible_neighbors       MapModel.covisible_neighbors mapmodel.py:269-273
 *   lm_ledger                    TransferLedger.as_dict devicestore.py:32-48
 */
#ifndef LM_B200_H
#define LM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum lm_status {
  LM_OK = 0,
  LM_ERR_INVALID_ARGUMENT = -1, /* InvalidArgumentError */
  LM_ERR_INVALID_STATE = -2,    /* InvalidStateError */
  LM_ERR_SLOT_CONFLICT = -3,    /* SlotConflictError */
  LM_ERR_CAPACITY = -4,         /* StoreCapacityError */
  LM_ERR_CUDA = -5,             /* CUDA runtime failure */
  LM_ERR_DEGENERATE = -6        /* DegenerateGeometryError */
} lm_status;

typedef struct lm_ctx lm_ctx;

typedef struct lm_map_caps {
  int32_t max_keyframes;        /* keyframe slots (covisibility is dense max_keyframes^2 int32) */
  int32_t max_keypoints;        /* keypoint pool over all keyframes */
  int32_t max_keypoints_per_kf; /* upper bound of one keyframe's keypoint count */
  int32_t max_points;           /* map point id space */
  int32_t obs_pool_entries;     /* observation pool (8 bytes per entry) */
  int32_t num_levels;           /* pyramid levels, <= 16 */
  double scale_factor;          /* pyramid scale factor (> 1) */
  int32_t min_covis_weight;     /* MapConfig.min_covis_weight */
  int32_t min_obs_keep;         /* MapConfig.min_obs_keep */
  /* StoreConfig ledger sizes */
  int32_t keypoint_record_bytes, descriptor_bytes, map_point_record_bytes, store_capacity;
} lm_map_caps;

typedef struct lm_match_cfg { /* MatchConfig config.py:22-30 */
  int32_t match_max_distance;
  double chi2_epi;
  int32_t level_window;
} lm_match_cfg;

typedef struct lm_gate_cfg { /* GateConfig config.py:13-19 */
  double cos_parallax_max, chi2_mono, scale_ratio_slack;
} lm_gate_cfg;

typedef struct lm_fuse_cfg { /* FuseConfig config.py:33-44 */
  int32_t match_max_distance;
  double fuse_radius, min_view_cos, dist_band_slack;
  int32_t level_window, n1, n2;
} lm_fuse_cfg;

typedef struct lm_cull_cfg { /* CullConfig config.py:63-72 (recent-point fields) */
  double found_ratio_min;
  int32_t probation_kfs, min_obs_graduate;
} lm_cull_cfg;

typedef struct lm_step_params {
  int32_t neighbor_count;
  int32_t do_cull, do_create, do_fuse; /* stage switches (1 = run) */
  int32_t processed_index;             /* pipeline._processed before this keyframe */
  lm_match_cfg match;
  lm_gate_cfg gate;
  lm_fuse_cfg fuse;
  lm_cull_cfg cull;
} lm_step_params;

#define LM_MAX_NEIGHBORS 64
#define LM_MAX_KF_SLOTS 8192 /* lm_map_caps.max_keyframes upper bound (shared-memory slot tables) */
#define LM_MAX_TARGETS 320

typedef struct lm_step_stats { /* CreationStats triangulation.py:49-60 + run_fusion counts */
  int32_t created, conflicts, degenerate;
  int32_t gate_parallax, gate_depth, gate_reprojection, gate_scale;
  int32_t n_degenerate_neighbors;
  int64_t degenerate_neighbors[LM_MAX_NEIGHBORS];
  int32_t n_neighbors;
  int64_t neighbors[LM_MAX_NEIGHBORS];
  int32_t n_targets;
  int32_t merged, observations_added, stale;
  int32_t culled;
  int64_t first_new_id; /* created ids are first_new_id .. first_new_id+created-1 */
  int32_t error;        /* nonzero: a device arena overflowed (lm_status code) */
  int32_t n_candidates; /* one-to-one search candidates over all neighbours */
  int64_t match_pairs;  /* P_elig: (unbound current, unbound level-window neighbour) pairs */
  int64_t fuse_bytes;   /* algorithmic fusion bytes, SURVEY.md 8(d) formula */
  int64_t fuse_passes, fuse_points, fuse_actions;
  int64_t apply_rounds;      /* deterministic-reservation rounds over all applies */
  int64_t fuse_cycles[16];   /* ns per fusion phase (%globaltimer): 0 targets, 2 fwd assemble,
                                3 fwd apply, 4 rev refresh, 5 rev geometry, 6 rev apply,
                                7 rev gather, 8 rev bound points, 9 apply reserve+check,
                                10 apply commit (plain), 11 apply merges, 12 apply compaction */
  int64_t rev_passes_acting;  /* reverse passes that produced at least one action */
  int64_t rev_passes_redo;    /* reverse-pass items re-evaluated after applies */
  int64_t fuse_bytes_rev;     /* algorithmic bytes of the reverse passes (part of fuse_bytes) */
  int64_t rev_mergeable;      /* acting passes none of whose (or earlier) items the previous apply touched */
  int64_t dbg[16];            /* diagnostic counters (meaning documented in bench.py) */
  /* borderline float compares (sides within 1e-10 relative, lm_math.cuh kFlipRel): the
   * decisions that could differ from the reference's (LAPACK SVD / NumPy log inputs).
   * [0] epipolar d^2 <= thr (k_match survivors), [1] triangulation degeneracy + creation
   * gates, [2] fusion projection / band / view-cos / radius gates (forward gather and the
   * speculative reverse evaluation), [3] rint ties of the fusion level prediction. */
  int64_t borderline[4];
  int64_t match_second_half;  /* pairs whose first 128 bits passed: the popcounts k_match executes
                                 are 4 * match_pairs + 4 * match_second_half */
} lm_step_stats;

typedef struct lm_candidate { /* MatchCandidate triangulation.py:41-46 */
  int64_t neighbor_kf_id;
  int32_t kp_index_current, kp_index_neighbor, distance, pad;
} lm_candidate;

#define LM_ACT_ADD 1
#define LM_ACT_MERGE 2
typedef struct lm_fuse_action { /* FuseAction fusion.py:29-35; existing_mp_id = -1 for None */
  int64_t target_kf_id, mp_id_projected;
  int32_t kp_index_hit, kind;
  int64_t existing_mp_id;
} lm_fuse_action;

typedef struct lm_ledger_t { /* TransferLedger devicestore.py:25-48 */
  int64_t persistent_bytes_up, naive_bytes_up;
  int64_t small_bytes_triangulation, small_bytes_fusion, small_transfer_events, evictions;
} lm_ledger_t;

typedef struct lm_map_sizes {
  int32_t n_kf_slots;  /* keyframe slots used (staged, live or dead) */
  int32_t n_points;    /* map point ids issued (next id) */
  int32_t n_keypoints; /* keypoint pool entries used */
  int32_t obs_used;    /* observation pool entries used */
  int32_t recent_n;    /* points under probation */
} lm_map_sizes;

/* ---- context / maps ---- */
int lm_version(void);
int lm_ctx_create(int32_t device, lm_ctx** out);
int lm_ctx_destroy(lm_ctx* ctx);
const char* lm_last_error(lm_ctx* ctx);
int lm_map_create(lm_ctx* ctx, const lm_map_caps* caps, int32_t* map_out);
int lm_map_reset(lm_ctx* ctx, int32_t map); /* back to an empty map, arenas kept */
int lm_map_destroy(lm_ctx* ctx, int32_t map); /* free the map's arenas (index not reused) */
int lm_map_sizes_get(lm_ctx* ctx, int32_t map, lm_map_sizes* out);
int lm_synchronize(lm_ctx* ctx);
/* programmatic dependent launch of the step kernels: 1 on, 0 off, -1 default (on for
 * single-map launch sequences); turn it off when several contexts step concurrently on one
 * device (a chain's parked successor CTAs hold SMs the other streams need) */
int lm_ctx_set_pdl(lm_ctx* ctx, int32_t mode);

/* ---- keyframes ---- */
/* Copy a keyframe into the map's pool without inserting it (not visible to any stage).
 * quat = (x,y,z,w) canonical unit quaternion, trans = world->camera translation,
 * cam = fx, fy, cx, cy, width, height. level: int64 per keypoint. bindings may be NULL
 * (all unbound); otherwise ids of live map points to register at insert. */
int lm_kf_stage(lm_ctx* ctx, int32_t map, int64_t kf_id, const double quat[4], const double trans[3],
                const double cam[6], int32_t n, const double* u, const double* v, const int64_t* level,
                const uint8_t* desc, const int64_t* bindings);
/* Binary keyframe record ("LMKF" v1), the ingest wire format replacing the reference's
 * JSON keyframe payload (service/schemas.py:111-126: KeyframePayload, hex descriptors) and
 * JSONL sequence lines (synth.py:376-439). Little-endian, 8-byte aligned:
 *   lm_kf_record_hdr (160 bytes), then double u[n], double v[n], uint8 level[n] padded to a
 *   multiple of 8, uint8 desc[32*n], and int64 bindings[n] when (flags & LM_REC_BINDINGS).
 * The record's pyramid (num_levels, scale_factor) must equal the map's. */
#define LM_REC_MAGIC 0x464B4D4Cu /* "LMKF" */
#define LM_REC_VERSION 1
#define LM_REC_BINDINGS 1u
typedef struct lm_kf_record_hdr {
  uint32_t magic;
  uint16_t version, flags;
  uint32_t n, header_bytes; /* keypoints; sizeof(lm_kf_record_hdr) */
  int64_t kf_id, frame_index;
  double quat[4];           /* x, y, z, w */
  double trans[3];          /* world -> camera */
  double fx, fy, cx, cy;
  int32_t width, height, num_levels, pad;
  double scale_factor;
  double reserved[2];
} lm_kf_record_hdr;
/* bytes of a record with n keypoints */
uint64_t lm_kf_record_bytes(int32_t n, uint32_t flags);
/* Validate one record and stage it like lm_kf_stage (kf_id_out may be NULL). */
int lm_kf_stage_record(lm_ctx* ctx, int32_t map, const void* record, uint64_t bytes, int64_t* kf_id_out);
/* Insert a staged keyframe into the map (insert_keyframe + upload_keyframe). */
int lm_kf_insert(lm_ctx* ctx, int32_t map, int64_t kf_id);
int lm_kf_kill(lm_ctx* ctx, int32_t map, int64_t kf_id); /* MapModel.kill_keyframe */
/* cull_keyframes culling.py:127-154 (redundancy by the per-level counter prefix,
 * is_redundant_fast 95-117 == is_redundant_baseline 60-92): candidates in ascending id order
 * (deduplicated, keyframe 0 and unknown/dead ids skipped), removal immediate (later
 * candidates see it), removed keyframes evicted from the store when resident. removed holds
 * up to n ids. */
typedef struct lm_kf_cull_cfg { /* CullConfig config.py:63-72 (keyframe fields) */
  double redundancy_ratio;
  int32_t min_redundant_observers, scale_tolerance_levels;
} lm_kf_cull_cfg;
int lm_cull_keyframes(lm_ctx* ctx, int32_t map, const int64_t* candidates, int32_t n, const lm_kf_cull_cfg* cfg,
                      int64_t* removed, int32_t* n_removed);

/* ---- the hot path ---- */
int lm_step(lm_ctx* ctx, int32_t map, int64_t kf_id, const lm_step_params* p, lm_step_stats* out);
/* Enqueue one step for each (map, keyframe) pair in one batched launch sequence. p points to
 * n lm_step_params, one per entry (each session keeps its own processed_index and stage
 * configs); a map may appear only once per batch. If out is NULL the call does not
 * synchronise (stats stay on the device until lm_step_stats_fetch, which also reports a
 * device-side error of the last step). */
int lm_step_batch(lm_ctx* ctx, int32_t n, const int32_t* maps, const int64_t* kf_ids, const lm_step_params* p,
                  lm_step_stats* out);
int lm_step_stats_fetch(lm_ctx* ctx, int32_t n, const int32_t* maps, lm_step_stats* out);
int lm_create_map_points(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t neighbor_count,
                         const lm_match_cfg* mc, const lm_gate_cfg* gc, lm_step_stats* out);
int lm_run_fusion(lm_ctx* ctx, int32_t map, int64_t kf_id, const lm_fuse_cfg* fc, lm_step_stats* out);
int lm_cull_recent(lm_ctx* ctx, int32_t map, int32_t processed_index, const lm_cull_cfg* cc, int32_t* culled);
/* cull_recent_map_points(model, recent, current_index, cfg) culling.py:28-59 in one call: the
 * probation list (ids, born) in, (removed ids, kept entries) out, each in list order; removed
 * and keep buffers hold n entries. An id naming no map point is skipped (neither removed nor
 * kept), as the reference skips `mp is None`; a point listed twice is LM_ERR_INVALID_ARGUMENT */
int lm_cull_recent_list(lm_ctx* ctx, int32_t map, int32_t processed_index, const lm_cull_cfg* cc, int32_t n,
                        const int64_t* ids, const int32_t* born, int64_t* removed, int32_t* n_removed,
                        int64_t* keep_ids, int32_t* keep_born, int32_t* n_keep);
int lm_search(lm_ctx* ctx, int32_t map, int64_t cur_kf, int64_t nbr_kf, const lm_match_cfg* mc,
              const uint8_t* unbound_cur, const uint8_t* unbound_nbr, lm_candidate* out, int32_t cap,
              int32_t* n_out);
int lm_fusion_targets(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t n1, int32_t n2, int64_t* out,
                      int32_t cap, int32_t* n_out);
int lm_fuse_pass(lm_ctx* ctx, int32_t map, const int64_t* point_ids, int32_t n, int64_t target_kf,
                 const lm_fuse_cfg* fc, lm_fuse_action* acts, int32_t act_cap, int32_t* n_act,
                 int64_t* visible, int32_t* n_vis);
int lm_apply_fusion(lm_ctx* ctx, int32_t map, const lm_fuse_action* acts, int32_t n, int32_t counts[3]);

/* ---- map bookkeeping (single-op kernels; the same device code the stages use) ---- */
int lm_mp_new(lm_ctx* ctx, int32_t map, const double pos[3], const uint8_t desc[32], int64_t first_kf,
              int64_t* id_out);
int lm_obs_add(lm_ctx* ctx, int32_t map, int64_t mp, int64_t kf, int32_t kp);
int lm_obs_erase(lm_ctx* ctx, int32_t map, int64_t mp, int64_t kf);
int lm_mp_kill(lm_ctx* ctx, int32_t map, int64_t mp);
int lm_mp_replace(lm_ctx* ctx, int32_t map, int64_t loser, int64_t winner, int32_t* migrated);
int lm_mp_set_counts(lm_ctx* ctx, int32_t map, int64_t mp, int32_t found, int32_t visible);
int lm_covisible_neighbors(lm_ctx* ctx, int32_t map, int64_t kf, int32_t n, int64_t* out, int32_t cap,
                           int32_t* n_out);
int lm_ledger(lm_ctx* ctx, int32_t map, lm_ledger_t* out);
/* explicit DeviceStore.record_neighbor_access / record_small_transfer (devicestore.py:80-101):
 * naive += naive_bytes; with small_events = 1 one small transfer of small_bytes (stage
 * "triangulation" if small_stage_triangulation, else "fusion") in both counters */
int lm_ledger_add(lm_ctx* ctx, int32_t map, int64_t naive_bytes, int32_t small_stage_triangulation,
                  int64_t small_bytes, int32_t small_events);
/* TransferLedger.per_stage_small_transfers: bytes of events first.. (at most cap), in order;
 * a negative entry b is a "triangulation" event of -b-1 bytes, others are "fusion" (the
 * stages log theirs: one forward pass + one per reverse pass). The first 65536 events of a
 * map are kept (the totals in lm_ledger are always exact). */
int lm_ledger_log(lm_ctx* ctx, int32_t map, int64_t first, int64_t* bytes, int32_t cap, int32_t* n_out);

/* ---- DeviceStore residency (devicestore.py:51-109) ----
 * lm_kf_insert is MapModel.insert_keyframe only; lm_kf_upload is DeviceStore.upload_keyframe
 * (residency + persistent ledger bytes; errors: already resident -> INVALID_STATE, capacity
 * -> CAPACITY). lm_step on a staged keyframe does both. A stage whose neighbours / fusion
 * targets include a non-resident keyframe fails with INVALID_STATE before touching the map
 * (record_neighbor_access devicestore.py:80-92). lm_kf_evict: evict_keyframe (not resident
 * -> INVALID_ARGUMENT). */
int lm_kf_upload(lm_ctx* ctx, int32_t map, int64_t kf_id);
int lm_kf_evict(lm_ctx* ctx, int32_t map, int64_t kf_id);
int lm_kf_resident(lm_ctx* ctx, int32_t map, int64_t kf_id, int32_t* resident, int32_t* count);
/* enforce = 0: the stages skip the residency check (the caller accounts residency in a store
 * of its own, e.g. the reference's DeviceStore); default 1 */
int lm_map_enforce_residency(lm_ctx* ctx, int32_t map, int32_t enforce);

/* ---- LBA write-back (localba.py:571-574 writes kf.pose and mp.position) ----
 * Poses and positions changed outside the hot path: the keyframe's R, t, C, P tables are
 * recomputed (same host code as staging) and the cached view geometry / hits of every
 * affected point invalidated, so the next stages see exactly the new values. */
int lm_kf_set_pose(lm_ctx* ctx, int32_t map, int64_t kf_id, const double quat[4], const double trans[3]);
int lm_mp_patch_positions(lm_ctx* ctx, int32_t map, int32_t n, const int64_t* ids, const double* pos);

/* ---- O(touched) reads for the MapModel facade ---- */
typedef struct lm_point_record { /* MapPoint mapmodel.py:65-77 */
  double pos[3];
  uint8_t rep[32];
  int64_t first_kf_id;
  int32_t alive, found, visible, nobs;
  int32_t counts[16]; /* scale_counts, num_levels used */
} lm_point_record;
/* one point (its representative descriptor refreshed if stale) + observations sorted by kf id */
int lm_mp_get(lm_ctx* ctx, int32_t map, int64_t mp, lm_point_record* out, int64_t* obs_kf, int32_t* obs_kp,
              int32_t obs_cap);
int lm_kf_bindings(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* out, int32_t cap, int32_t* n_out);
int lm_mp_alive(lm_ctx* ctx, int32_t map, int32_t n, const int64_t* ids, uint8_t* out); /* MapPoint.alive of n ids */
int lm_bound_points(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* out, int32_t cap, int32_t* n_out);
/* nonzero covisibility entries of one keyframe (any order): CovisibilityGraph adjacency */
int lm_covis_row(lm_ctx* ctx, int32_t map, int64_t kf_id, int64_t* kf_ids, int32_t* weights, int32_t cap,
                 int32_t* n_out);

/* ---- snapshot import (per-step parity from a reference state; SURVEY.md 5 checkpoint row) ----
 * Keyframes in insertion (kf id) order; keypoint arrays concatenated (kp_n per keyframe).
 * Dead keyframes carry no bindings. Points are ids 0..n_points-1 (dead ones included).
 * The map must be empty (fresh or lm_map_reset). */
typedef struct lm_snapshot {
  int32_t n_kf;
  const int64_t* kf_id;
  const uint8_t* kf_alive;
  const uint8_t* kf_resident; /* may be NULL: none resident */
  const double* quat;         /* 4 per keyframe (x, y, z, w) */
  const double* trans;        /* 3 per keyframe */
  const double* cam;          /* 6 per keyframe: fx, fy, cx, cy, width, height */
  const int32_t* kp_n;
  const double* u;
  const double* v;
  const int64_t* level;
  const uint8_t* desc;     /* 32 per keypoint */
  const int64_t* bindings; /* -1 = unbound */
  int32_t n_points;
  const double* pos;       /* 3 per point */
  const uint8_t* rep;      /* 32 per point */
  const uint8_t* alive;
  const int32_t* found;
  const int32_t* visible;
  const int64_t* first_kf; /* may be NULL */
  int32_t n_recent;        /* probation list (culling.RecentPoint) */
  const int64_t* recent_id;
  const int32_t* recent_born;
  lm_ledger_t ledger;
} lm_snapshot;
int lm_import_snapshot(lm_ctx* ctx, int32_t map, const lm_snapshot* snapshot);

/* ---- device audit (MapModel.audit mapmodel.py:304-353) ----
 * codes: 1 dead point keeps observations (mp); 2 point observes a dead keyframe (mp, kf_a);
 * 3 binding mismatch (mp, kf_a, kp); 4 scale_counts mismatch (mp); 5 scale_counts sum
 * mismatch (mp); 6 slot bound to a dead point (kf_a, kp, mp); 7 slot not in the point's
 * observations (kf_a, kp, mp); 8 covisibility weight mismatch (kf_a, kf_b). Order unspecified;
 * *n_out = total found (records beyond cap are dropped). */
typedef struct lm_audit_record {
  int32_t code, kp;
  int64_t mp, kf_a, kf_b;
} lm_audit_record;
int lm_audit(lm_ctx* ctx, int32_t map, lm_audit_record* out, int32_t cap, int32_t* n_out);
/* fault injection for audit tests: what 0 = counter cell (mp a, level b) += delta; what 1 =
 * covisibility (kf a, kf b) += delta, both directions (CovisibilityGraph.bump) */
int lm_debug_corrupt(lm_ctx* ctx, int32_t map, int32_t what, int64_t a, int64_t b, int32_t delta);

/* ---- state export (parity, snapshots) ---- */
/* keyframe table: per slot kf_id, state (1 staged, 2 live, 3 dead), kp_off, kp_n */
int lm_export_keyframes(lm_ctx* ctx, int32_t map, int64_t* kf_id, int32_t* state, int32_t* kp_off,
                        int32_t* kp_n, int32_t cap, int32_t* n_out);
int lm_export_bindings(lm_ctx* ctx, int32_t map, int32_t* bind, int32_t cap); /* whole keypoint pool */
/* points 0..n-1: pos[3n], rep[32n], alive[n], found[n], visible[n], nobs[n], counts[n*L];
 * observations flattened in id order (each point's list sorted by kf id): obs_kf[], obs_kp[]. */
int lm_export_points(lm_ctx* ctx, int32_t map, int32_t n, double* pos, uint8_t* rep, uint8_t* alive,
                     int32_t* found, int32_t* visible, int32_t* nobs, int32_t* counts, int64_t* obs_kf,
                     int32_t* obs_kp, int32_t obs_cap);
int lm_export_covis(lm_ctx* ctx, int32_t map, int32_t* w, int32_t cap); /* dense slot x slot */
int lm_recent_export(lm_ctx* ctx, int32_t map, int64_t* ids, int32_t* born, int32_t cap, int32_t* n_out);
int lm_recent_import(lm_ctx* ctx, int32_t map, const int64_t* ids, const int32_t* born, int32_t n);

/* ---- measurement ---- */
/* Rewind a map to "all keyframes staged, nothing inserted": keeps the keyframe pool (no
 * host transfer) so a sequence can be replayed with device-resident inputs. */
int lm_map_rewind(lm_ctx* ctx, int32_t map);
int lm_timer_start(lm_ctx* ctx);                 /* CUDA event on the context stream */
int lm_timer_stop(lm_ctx* ctx, float* ms);       /* event + synchronize, elapsed since start */
/* Timing across two contexts (streams) of one device: start on ctx (other waits for it),
 * stop = the later of both streams. */
int lm_timer_start_joint(lm_ctx* ctx, lm_ctx* other);
int lm_timer_stop_joint(lm_ctx* ctx, lm_ctx* other, float* ms);
/* the same over n contexts (start on ctxs[0], stop = the latest stream) */
int lm_timer_start_multi(lm_ctx* const* ctxs, int32_t n);
int lm_timer_stop_multi(lm_ctx* const* ctxs, int32_t n, float* ms);
int lm_flush_l2(lm_ctx* ctx, int64_t bytes);     /* write a scratch buffer larger than L2 */
int64_t lm_launch_count(lm_ctx* ctx);
/* Running totals since map creation/reset/rewind (first_new_id holds the step count). */
int lm_totals_fetch(lm_ctx* ctx, int32_t map, lm_step_stats* out);            /* kernels launched by this context so far */
/* Per-stage CUDA-event timing of the step kernels (stage order: begin+insert, cull, select,
 * prep, match, tri, commit, fuse_targets, fuse_geo, fuse_gather, fuse_apply, fuse_refresh,
 * fuse_rev+end). Enabling adds one event per stage boundary per step and turns on the
 * kernels' in-step phase timers (lm_step_stats fuse_cycles / dbg time fields; device-wide),
 * which read 0 otherwise. */
int lm_profile_enable(lm_ctx* ctx, int32_t on);
int lm_profile_read(lm_ctx* ctx, double ms[16], int64_t launches[16]); /* sums, then clears */
/* Sustained __popc throughput of this device (popc32 results per second). */
int lm_bench_popc(lm_ctx* ctx, double* popc_per_s);

/* ---- host-side math, exported for CPU parity tests (no GPU needed) ---- */
int lm_host_fundamental(const double qa[4], const double ta[3], const double qb[4], const double tb[3],
                        const double cam_a[4], const double cam_b[4], double F[9]);
int lm_host_projection(const double quat[4], const double trans[3], const double cam[4], double R[9],
                       double C[3], double P[12]);
int lm_host_triangulate(const double Pa[12], const double Pb[12], const double Ca[3], const double Cb[3],
                        const double pix[4], double X[3]);

#ifdef __cplusplus
}
#endif
#endif /* LM_B200_H */
