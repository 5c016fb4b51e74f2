/*
 * sparrow.h -- C-ABI of the B200-native Sparrow hot path (libsparrow.so).
 *
 * Plain pointers and sizes only; no torch types.  Device pointers are CUDA
 * global-memory pointers on the handle's device; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Every entry point returns an SpStatus; the
 * thread-local message of the last failure is sp_last_error().
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/color_rl):
 *
 *   sp_cast_rays        kernels/__init__.py:62-76 -> kernels/_cy.pyx:19-106
 *   sp_disc_collides    kernels/__init__.py:79-86 -> kernels/_cy.pyx:109-158
 *   sp_env_create       vecenv.py:61-80 (VecEnv.__init__) + sim/core.py:47-110
 *                       (SimBatch.__init__; map stacking core.py:62-71)
 *   sp_env_reset_all    vecenv.py:84-92 (VecEnv.reset_all) -> core.py:114-161
 *   sp_env_step         vecenv.py:94-116 (VecEnv.step_batch) -> core.py:165-219
 *   sp_env_step_host    the same with host buffers (numpy in/out contract)
 *                       (SimBatch.step_all) incl. fused auto-reset core.py:114-161
 *   sp_env_stats_*      vecenv.py:120-141 (snapshot_stats, first_episode_outcomes)
 *   sp_env_read_state   sim/core.py:88-108 SoA attributes (read-only views)
 *   sp_env_write_state  test-only pose placement (tests/test_env.py:37-42 place())
 *   sp_env_reset_lanes  sim/core.py:114-161 (SimBatch.reset_lane, stream kept)
 *   sp_env_scan         sim/core.py:223-235 (SimBatch._scan) on caller poses
 *   sp_rb_create        replay.py:31-43 (ReplayBuffer.__init__)
 *   sp_rb_append        replay.py:48-67 (append_batch)
 *   sp_rb_sample        replay.py:69-79 (sample)
 *   sp_rb_size          replay.py:45-46 (__len__)
 *   sp_rb_gather        replay.py:81-87 (snapshot: rows in storage order)
 *   sp_random_actions   bench.py:97-105 (random policy actions), on device
 *   sp_philox_fill      asl/vem.py:57-66 draws (rng.random / rng.integers), on device
 *   sp_adam_step        net.py:141-161 adam_step, fused over all tensors, on device
 *   sp_ddqn_update      ddqn.py:54-77 DdqnLearner.update (targets, backprop, Adam), on device
 *   sp_actor_select     asl/loops.py:57-60 + net.py:77-80 + asl/vem.py:38-66: forward, VEM
 *                       epsilons and epsilon-greedy selection in one launch
 */
#ifndef SPARROW_H_
#define SPARROW_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SP_OK = 0,
  SP_EINVAL = 1,        /* ValueError: bad shape/config (core.py:56-59, vecenv.py:66-67) */
  SP_EACTION = 2,       /* ValueError: action index out of range (core.py:169-170) */
  SP_EEPISODE = 3,      /* EpisodeTerminated (core.py:35, 171-174) */
  SP_EMAP = 4,          /* MapError: shapes differ / no spawn pose (core.py:63-66, 144-147) */
  SP_ENOTREADY = 5,     /* BufferNotReady (replay.py:19, 73-75) */
  SP_ECUDA = 6,         /* CUDA runtime failure */
  SP_ENOMEM = 7
} SpStatus;

#define SP_MAX_ACTIONS 15 /* action codes are 4-bit; 15 marks the (0,0) delay filler */
#define SP_MAX_DELAY 64   /* params.py:20 MAX_CONTROL_DELAY */

/* EnvConfig + LidarConfig (sim/params.py:124-151) */
typedef struct {
  int32_t n_beams;             /* LidarConfig.n_beams */
  double max_range_cm;         /* LidarConfig.max_range_cm */
  double robot_radius_cm;      /* EnvConfig.robot_radius_cm */
  int32_t timeout_steps;       /* EnvConfig.timeout_steps */
  double proximity_cm;         /* EnvConfig.obstacle_penalty_range_cm */
  int32_t n_actions;           /* len(EnvConfig.action_table) <= SP_MAX_ACTIONS */
  double action_table[2 * SP_MAX_ACTIONS]; /* (v_linear, v_angular) pairs */
  int32_t spawn_attempts;      /* EnvConfig.spawn_attempts */
  int32_t auto_reset;          /* VecEnv(auto_reset=...) */
  const double* beam_offsets;  /* host, n_beams: LidarConfig.beam_offsets() */
} SpConfig;

/* One occupancy map (sim/gridmap.py GridMap); all maps of an env share shape. */
typedef struct {
  int32_t n_rows, n_cols;      /* grid shape (H, W) */
  double cell_cm;              /* cell_size_cm */
  const uint8_t* occupancy;    /* host, H*W row-major [iy][ix], nonzero = occupied */
  double goal_x, goal_y, goal_radius;
  double spawn[4];             /* x0, y0, x1, y1 */
  double planning_dist;        /* EnvConfig.planning_dist(map) */
} SpMapDesc;

/* DiversityRanges (params.py:55-121), one per lane or one shared. */
typedef struct {
  double k[2], dt[2];
  int32_t delay[2];            /* inclusive */
  double vmax_linear[2], vmax_angular[2], noise_std[2];
} SpRanges;

typedef struct SpEnv SpEnv;
typedef struct SpReplay SpReplay;

const char* sp_last_error(void);
int sp_version(void);
int sp_device_info(int device, int* n_sm, int* smem_optin_bytes, int* cc_major, int* cc_minor);

/* ---- environment ------------------------------------------------------- */
int sp_env_create(const SpConfig* cfg, const SpMapDesc* maps, int32_t n_maps, int64_t n_envs,
                  const int32_t* map_index /* host, n_envs, or NULL = (offset+i) % n_maps */,
                  const SpRanges* ranges, int64_t n_ranges /* 1 or n_envs */,
                  int64_t env_id_offset, int device, SpEnv** out);
int sp_env_destroy(SpEnv* env);
int sp_env_reset_all(SpEnv* env, uint64_t seed, float* states /* dev (N, 5+R) */, void* stream);
/* states and store_states must not overlap (with auto-reset an env's two scans
 * park their LiDAR noise in different rows): SP_EINVAL otherwise. */
int sp_env_step(SpEnv* env, const int64_t* actions /* dev (N) */, float* states,
                float* store_states, double* rewards, uint8_t* dones, uint8_t* truncated,
                int8_t* events, void* stream);
/* Recording (parity / inspection; off by default, costs nothing when off):
 * every following reset_all / step / reset_lanes also writes, per caller row
 * and beam (dev int32/f64 [N][R], row-major, NULL = not recorded),
 *   hit_store  the occupied cell iy*W+ix each ray of the post-step scan (the
 *              store_states rows) stopped in, -1 at max range / grid exit;
 *   hit_state  the same for the scan behind the returned states rows (the
 *              fresh-spawn scan of an env that reset, else the post-step one);
 *   scan_state that scan's noisy clipped range in cm: SimBatch.last_scan
 *              (sim/core.py:97, 237-241).
 * The bit-exact hit-cell parity tests read these against the oracle's DDA. */
int sp_env_set_recording(SpEnv* env, int32_t* hit_store, int32_t* hit_state,
                         double* scan_state);
/* Host-buffer step: the reference's numpy step_batch contract (vecenv.py:94-116)
 * for callers holding host memory.  h_actions: N int64; h_out: one contiguous
 * block of sp_env_host_out_bytes(env) bytes laid out as
 *   rewards f64[N] | states f32[N][5+R] | store_states f32[N][5+R] |
 *   dones u8[N] | truncated u8[N] | events i8[N].
 * The H2D copy of the actions, the fused step, the D2H copy of the block
 * (device staging owned by the handle); returns after everything synchronized.
 * The actions are checked on the host while their copy is in flight: one
 * outside [0, n_actions) returns SP_EACTION before anything is launched, so
 * nothing steps (core.py:169-170).
 * From 16,384 envs (default map assignment) the step runs as row parts (two:
 * a quarter of the rows, then the rest): part
 * p's launch, then its obs rows' copy on a second stream while part p + 1
 * steps (SPARROW_HOST_PARTS sets the count, 1 = one launch and one copy on
 * `stream`).  Page-locked host memory lets the copies run at full PCIe
 * bandwidth.  Invalid actions are reported by sp_env_check as after sp_env_step. */
int64_t sp_env_host_out_bytes(SpEnv* env);
int sp_env_step_host(SpEnv* env, const int64_t* h_actions, void* h_out, void* stream);
/* Sticky device error word from the last step (SP_OK if none); syncs `stream`. */
int sp_env_check(SpEnv* env, void* stream, int64_t* err_env);
/* 1 if any lane waits for a reset (auto_reset=0 path; core.py:171-174); syncs. */
int sp_env_any_needs_reset(SpEnv* env, void* stream, int* any);

/* per-copy stats in external env order (host arrays of n_envs) */
int sp_env_stats_read(SpEnv* env, int64_t* episodes, int64_t* arrivals, double* return_sum,
                      int8_t* first_event, double* first_return, int64_t* first_steps,
                      void* stream);
/* last <=256 finished-episode returns in (step, env) order (vecenv.py:79,105) */
int sp_env_recent_returns(SpEnv* env, double* out256, int32_t* n_out, void* stream);
/* The same with each return's order key (step << 32) | global env id, so the
 * shards of a multi-GPU run merge into the single-process deque (dist.py). */
int sp_env_recent_returns_keyed(SpEnv* env, double* out256, uint64_t* keys256, int32_t* n_out,
                                void* stream);
int sp_env_stats_reset(SpEnv* env, int clear_recent, void* stream);
/* device totals {episodes, arrivals, return_sum} as 3 doubles (all-reduce payload) */
int sp_env_stats_totals(SpEnv* env, double* dev_out3, void* stream);
/* Lanes whose first episode since reset_all has not ended (first_event < 0;
 * the latch behind first_episode_outcomes, vecenv.py:134-141): a device
 * count and one 8-byte read; synchronizes `stream`. */
int sp_env_first_pending(SpEnv* env, int64_t* host_count, void* stream);

/* read one SoA field, external env order, into a host array of n_envs doubles.
 * field: 0 x, 1 y, 2 heading, 3 v_linear, 4 v_angular, 5 start_x, 6 start_y,
 * 7 k, 8 dt, 9 delay, 10 vmax_linear, 11 vmax_angular, 12 noise_std,
 * 13 step_count, 14 needs_reset, 15 rng_ctr, 16 episode_return */
int sp_env_read_state(SpEnv* env, int field, double* host_out, void* stream);
/* overwrite one pose field (ids 0-6 above, 17 start_cos, 18 start_sin) from a
 * host array (external order) -- the reference tests' place() (test_env.py:37-42) */
int sp_env_write_state(SpEnv* env, int field, const double* host_in, void* stream);
/* The delay FIFO of every lane (SimBatch._pending, sim/core.py:106, 156,
 * 176-182) as host u64 [N][4] in caller row order: a shift register of 4-bit
 * action codes, nibble q of the 256-bit word = the action issued q steps ago
 * (q = 0 newest), code 15 = the (0, 0) filler a reset queues; the lane's
 * control delay d says how many of the nibbles are pending (q < d). */
int sp_env_read_fifo(SpEnv* env, uint64_t* host_out, void* stream);
/* SimBatch.reset_lane (core.py:114-161) for the lanes with mask[i] != 0 (device,
 * external order), continuing each lane's stream; writes their rows of states. */
int sp_env_reset_lanes(SpEnv* env, const uint8_t* mask, float* states, void* stream);
int sp_env_map_info(SpEnv* env, int64_t* slot_of_env /* host n_envs, may be NULL */,
                    int64_t* smem_bytes, int32_t* threads_per_cta, int32_t* ctas);
/* Launch partition (diagnostics): the step kernel's CTA slot cuts (host
 * ctas+1, may be NULL) and the SM cycles each CTA took in the last step (host
 * ctas, may be NULL).  Synchronizes the device. */
int sp_env_launch_info(SpEnv* env, int64_t* cuts, uint32_t* cta_cycles);

/* LiDAR scan with the fused step's marcher on caller poses (no noise).
 * Queries must be grouped by map: query q of map m lies in
 * [query_offsets[m], query_offsets[m+1]).
 * ranges[q*R + j], hit_cell[q*R + j] = iy*W+ix of the stopping occupied cell or -1. */
int sp_env_scan(SpEnv* env, int64_t n,
                const int64_t* query_offsets /* host n_maps+1; queries sorted by map */,
                const double* x /* dev */, const double* y, const double* heading,
                double* ranges /* dev n*R */, int32_t* hit_cell /* dev n*R or NULL */,
                void* stream);

/* ---- op-level plugin seam (kernels/_cy.pyx signature), device in/out ---- */
int sp_cast_rays(const uint8_t* occ, const double* edt, int64_t n_maps, int64_t height,
                 int64_t width, const int64_t* map_idx, const double* px, const double* py,
                 const double* dirx, const double* diry, int64_t n, double cell,
                 double max_range, double* out, void* stream);
int sp_disc_collides(const uint8_t* occ, int64_t n_maps, int64_t height, int64_t width,
                     const int64_t* map_idx, const double* px, const double* py,
                     const double* radius, int64_t n, double cell, uint8_t* out, void* stream);

/* ---- replay ring (replay.py) -------------------------------------------- */
int sp_rb_create(int64_t capacity, int32_t state_dim, int device, SpReplay** out);
int sp_rb_destroy(SpReplay* rb);
/* rewards: reward_is_f64 ? double* : float*.  n <= capacity. */
int sp_rb_append(SpReplay* rb, const float* states, const int64_t* actions, const void* rewards,
                 int reward_is_f64, const float* next_states, const uint8_t* dones, int64_t n,
                 void* stream);
/* uniform with replacement over [0, size): idx_i = mulhi64(philox(seed, ctr+i, stream_id, 2), size) */
int sp_rb_sample(SpReplay* rb, int64_t batch, uint64_t seed, uint32_t stream_id, uint64_t ctr,
                 float* states, int64_t* actions, float* rewards, float* next_states,
                 uint8_t* dones, int64_t* idx_out, void* stream);
/* sample with the fill level and the first Philox block read from device memory
 * (*d_ctr, advanced by batch on the device afterwards): the same draws as
 * sp_rb_sample(..., ctr = *d_ctr, ...), but CUDA-graph capturable.  The caller
 * gates on sp_rb_size >= batch (BufferNotReady) and orders it after appends. */
int sp_rb_sample_dev(SpReplay* rb, int64_t batch, uint64_t seed, uint32_t stream_id,
                     uint64_t* d_ctr, float* states, int64_t* actions, float* rewards,
                     float* next_states, uint8_t* dones, int64_t* idx_out, void* stream);
int sp_rb_size(SpReplay* rb, int64_t* size, int64_t* cursor);
/* gather rows [0, size) in storage order */
int sp_rb_gather(SpReplay* rb, float* states, int64_t* actions, float* rewards,
                 float* next_states, uint8_t* dones, void* stream);

/* ---- benchmark helpers ----------------------------------------------------- */
/* Philox stream draws on device (DESIGN.md RNG contract), blocks ctr0 .. ctr0+n-1 of
 * (seed, lane, tag): kind 0 -> double out[i] = uniform(lo, hi); kind 1 -> int64
 * out[i] = integers(lo, hi).  The VEM epsilon-greedy draws (asl/vem.py:57-66). */
int sp_philox_fill(int64_t n, uint64_t seed, uint32_t lane, uint32_t tag, uint64_t ctr0,
                   int kind, double lo, double hi, void* out, void* stream);
/* actions[i] = integers(0, n_actions) from block `step` of (seed, env_id0 + i, tag 1) */
int sp_random_actions(int64_t n, uint64_t seed, int64_t env_id0, int64_t step, int32_t n_actions,
                      int64_t* actions, void* stream);

/* ---- learner side ------------------------------------- */
#define SP_ADAM_MAX 16
/* Bias-corrected Adam over n_tensors fp32 device tensors in one launch; replaces
 * net.py:141-161 (_adam_update / adam_step), same op order and fp32 roundings.
 * params/grads/m/v: host arrays of device pointers; numels: host array.
 * t = step_dev ? *step_dev + 1 (then *step_dev += 1 on device) : step_host.
 * gate (nullable device scalar, e.g. the loss): the step applies only if it is
 * finite, so a diverged update leaves every tensor untouched (ddqn.py:66-71). */
int sp_adam_step(int n_tensors, float* const* params, const float* const* grads, float* const* m,
                 float* const* v, const int64_t* numels, double* step_dev, int64_t step_host,
                 const float* gate, double lr, double beta1, double beta2, double eps,
                 void* stream);

/* The Q-net of net.py: sizes {D0, H1, H2, A}; W[l] row-major (fan_in, fan_out)
 * fp32 device arrays, b[l] (fan_out). */
typedef struct SpMlp {
  int32_t sizes[4];
  float* W[3];
  float* b[3];
} SpMlp;

/* scratch (floats) sp_ddqn_update needs for a batch of `batch` rows, or -1 when the
 * layer sizes / batch exceed the fused kernels (shared-memory staging limits) */
int64_t sp_ddqn_scratch_floats(const int32_t* sizes, int64_t batch);
/* One double-DQN update in three launches (row-parallel forward/deltas,
 * parameter-parallel gradient + gated Adam, step tick); replaces ddqn.py:54-77 (DdqnLearner.
 * update: compute_targets :38-51, net.backward :88-115, adam_step net.py:151-161).
 * Batch columns are device arrays (s, s2: (batch, D0) f32; a i64; r f32; d u8).
 * m/v: the six Adam moment tensors in W1 W2 W3 b1 b2 b3 order; *step_dev is the
 * Adam step count (incremented on device when the update applies).  The update
 * applies only if the loss is finite (ddqn.py:66-71); stats_out (device, 2 f32)
 * receives {mean Huber loss, mean |td|}.  Requires D0 <= 128, H1, H2 <= 256,
 * A <= 16, 16-byte aligned weights and sp_ddqn_scratch_floats(...) >= 0 (the
 * three staged weight matrices fit in shared memory: e.g. [32|37,256,128,5]).
 * The target net is read only. */
/* VemSchedule (asl/vem.py:19-35) */
typedef struct {
  int64_t n_envs, or_init, or_final, decay_steps;
  double e_min, e_max;
} SpVem;

/* The actor's input to an env step in one launch (asl/loops.py:57-60):
 * Q = MLP(states) (net.py:77-80), the VEM epsilon of copy env0 + i at t_step
 * computed on the device (vem.py:38-54), epsilon-greedy selection
 * (vem.py:57-66) drawing explore tests from blocks ctr .. ctr+n-1 and random
 * actions from ctr+n .. ctr+2n-1 of Philox stream (seed, lane, tag) -- the
 * caller advances its counter by 2n.  actions: dev int64 [n]; q_out: dev f32
 * [n][A] or NULL.  Weights: 16-byte aligned fp32 device tensors, layer
 * sizes D0 <= 64, H1, H2 <= 256, A <= 16, each matrix a multiple of 4 floats. */
int sp_actor_select(const SpMlp* net, const float* states, int64_t n, int64_t env0,
                    const SpVem* vem, int64_t t_step, uint64_t seed, uint32_t lane, uint32_t tag,
                    uint64_t ctr, int64_t* actions, float* q_out, void* stream);

int sp_ddqn_update(const SpMlp* online, const SpMlp* target, const float* s, const int64_t* a,
                   const float* r, const float* s2, const uint8_t* d, int64_t batch, float gamma,
                   float* const* m, float* const* v, double* step_dev, double lr, double beta1,
                   double beta2, double eps, float* scratch, int64_t scratch_floats,
                   float* stats_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARROW_H_ */
