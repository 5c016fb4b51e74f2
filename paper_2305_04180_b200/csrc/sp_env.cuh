// sp_env.cuh -- device-side data layout of one Sparrow environment batch.
#pragma once
#include "sp_common.cuh"

// Launch shape: SP_CTAS_PER_SM resident CTAs of SP_CTA_THREADS threads (one
// 768-thread CTA per SM by default; a build with SP_CTAS_PER_SM=2 gives each
// of two CTAs its own copy of its map's tables).
#ifndef SP_CTAS_PER_SM
#define SP_CTAS_PER_SM 1
#endif
#ifndef SP_CTA_THREADS
#define SP_CTA_THREADS (768 / SP_CTAS_PER_SM)
#endif

#ifndef SP_PLAN_MAX
#define SP_PLAN_MAX 296  // CTAs whose slot range rides in the kernel parameters
#endif

namespace sp {

// Per-map constants (gridmap.py GridMap fields used by core.py:81-86, 133).
struct MapConst {
  double goal_x, goal_y, goal_r, plan_dist;
  double spawn[4];
  double inv_plan;  // 1 / plan_dist (correctly rounded; quotients use div_by)
};

// Byte offsets (from the dynamic shared-memory base) of the chunk's arrays
// (Chunk in sp_env.cu): SlotRec rec[slots] (80 B) | double retp[cap], part[cap]
// | u32 gid[slots] | i32 reg[slots], hwrite[slots] | i32 xslot[cap] |
// i32 ctl[24] | i32 rowi[cap], send[cap] | u16 list[8 slots] | u8 wmode[cap],
// evs[cap] | u8 prox[slots].  Kernel parameters, so every array address is
// one constant-bank operand away (nothing to keep in registers).
enum ChunkField { CF_REC, CF_RETP, CF_PART, CF_GID, CF_REG, CF_HWRITE, CF_XSLOT, CF_CTL, CF_ROWI,
                  CF_SEND, CF_LIST, CF_WMODE, CF_EVS, CF_PROX, CF_END, CF_N };
__host__ __device__ inline void chunk_offsets(uint32_t base, int cap, int slots, uint32_t* o) {
  const uint32_t c = (uint32_t)cap, s = (uint32_t)slots;
  o[CF_REC] = base;
  o[CF_RETP] = o[CF_REC] + 80u * s;
  o[CF_PART] = o[CF_RETP] + 8u * c;
  o[CF_GID] = o[CF_PART] + 8u * c;
  o[CF_REG] = o[CF_GID] + 4u * s;
  o[CF_HWRITE] = o[CF_REG] + 4u * s;
  o[CF_XSLOT] = o[CF_HWRITE] + 4u * s;
  o[CF_CTL] = o[CF_XSLOT] + 4u * c;
  o[CF_ROWI] = o[CF_CTL] + 96u;
  o[CF_SEND] = o[CF_ROWI] + 4u * c;
  o[CF_LIST] = o[CF_SEND] + 4u * c;
  o[CF_WMODE] = o[CF_LIST] + 16u * s;
  o[CF_EVS] = o[CF_WMODE] + c;
  o[CF_PROX] = o[CF_EVS] + c;
  o[CF_END] = o[CF_PROX] + s;
}

// Everything the step kernel reads, by value (kernel parameter).
struct EnvDev {
  int64_t n;              // lanes (slots)
  int32_t R, D;           // beams, obs dim = 5 + R
  int32_t H, W, Hb, Wb, WW;  // grid, march-table grid (= grid: per cell), 32-bit words per bitmap row
  int32_t n_maps;
  double cell, inv_cell, max_range, radius, proximity;
  int32_t timeout, spawn_attempts, auto_reset, n_actions;
  int32_t need_k;         // cell-box radius that proves "no disc collision" (ceil(radius / cell))
  uint32_t blk_bytes;     // per-map march (cell) table bytes (16-byte padded)
  uint32_t bits_bytes;    // per-map bitmap bytes
  uint32_t map_bytes;     // blk_bytes + bits_bytes
  double action_v[SP_MAX_ACTIONS + 1], action_w[SP_MAX_ACTIONS + 1];  // code 15 = (0, 0)
  const uint8_t* maps;    // n_maps * map_bytes: [blk | bits]
  const MapConst* mconst; // n_maps
  const int64_t* map_off; // n_maps + 1 slot ranges (slots are map-major)
  const double2* beam_cs; // R: (cos, sin) of LidarConfig.beam_offsets()
  // SoA state, slot order (core.py:88-108)
  double *x, *y, *h, *vl, *va, *ret;
  double *sx, *sy, *c0, *s0, *pk, *pdt, *pvl, *pva, *psig;
  uint64_t* hist;         // 4 words per lane: hist[w * n + s]; 4-bit action codes
  uint64_t* ctr;          // Philox block counter per lane
  int32_t *step, *delay;
  uint8_t* needs_reset;
  uint64_t* qhist;        // n: per beam group, the step levels of the lane's last scan (8 x u8)
  const double* ranges;   // 12 doubles per lane (or shared when ranges_shared)
  int32_t ranges_shared;
  const int64_t* env_of_slot;
  int64_t env_id_offset;
  uint64_t seed;
  // per-copy stats (vecenv.py:33-41, 76-80), slot order
  int64_t *episodes, *arrivals;
  double* return_sum;
  int8_t* first_event;
  double* first_ret;
  int32_t* first_steps;
  double* rec_ret;        // recent-returns ring (vecenv.py:79)
  uint64_t* rec_key;      // (step << 32) | env row, for deterministic ordering
  unsigned long long* rec_count;
  uint64_t rec_cap;
  int32_t* err;           // [0] status, [1] env row
  uint32_t* cta_cyc;      // grid: SM cycles each CTA took in the last MODE_STEP launch
  // launch geometry
  const int64_t* cta_begin;  // grid + 1 slot boundaries (map-aligned when possible)
  int32_t chunk_cap;      // envs per CTA chunk (<= threads per CTA)
  int32_t slot_cap;       // scan slots per chunk: chunk_cap + extra post-reset slots
  int32_t nb, nb_shift;   // Philox blocks of LiDAR noise per scan (ceil(R/4)); log2 or -1
  double inv_max_range;
  uint32_t off_beam, off_bar, off_chunk;  // smem offsets
  uint32_t co[CF_N];      // chunk array offsets (chunk_offsets)
  int32_t smem_maps;      // 1: tables staged in shared memory via TMA bulk copy
  int32_t refill_min;     // ray queue: refill a warp once this many lanes idle
  int32_t prenoise;       // LiDAR noise blocks each idle thread draws during phase A
  int32_t late_resets;    // 1: auto-resets by the reset warp (reset_late), 0: inline
  int32_t gshift;         // beams per dispatch group = 2^gshift (<= 8 groups per scan)
  int32_t n_groups;       // groups per scan: ceil(R / 2^gshift)
  uint64_t d_magic;       // ceil(2^40 / D): f / D for f < 2^21 (row writes)
  // caller row of a slot without the env_of_slot load, for the default map
  // assignment map = (env_id_offset + row) % n_maps: slot s of map m is row
  // i0(m) + (s - map_off[m]) * n_maps, i0(m) = (m - off_mod) mod n_maps
  int32_t row_affine;
  int32_t off_mod;        // env_id_offset % n_maps
  // launch plan in the parameters (constant bank): a CTA starts without a
  // global-memory round trip.  plan_n == 0: read cta_begin / map_off instead
  int32_t plan_n;
  int32_t plan_begin[SP_PLAN_MAX + 1];  // slot range of CTA b: [begin[b], end[b])
  int32_t plan_end[SP_PLAN_MAX];        // = begin[b + 1], except in a part plan (row parts)
  int32_t plan_mstart[SP_PLAN_MAX];     // map_off[map of the CTA's first slot]
  int32_t plan_mend[SP_PLAN_MAX];       // map_off[that map + 1]
  int16_t plan_map[SP_PLAN_MAX];        // that map
};

enum { MODE_STEP = 0, MODE_RESET_ALL = 1, MODE_RESET_LANES = 2 };

struct StepArgs {
  int32_t mode;
  uint64_t step_index;
  const int64_t* actions;  // external order
  const uint8_t* reset_mask;  // MODE_RESET_LANES: external order
  float* states;           // (N, D) post-reset obs
  float* store_states;     // (N, D) pre-reset s'
  double* rewards;
  uint8_t* dones;
  uint8_t* truncated;
  int8_t* events;
  // optional recording (sp_env_set_recording; null = off, the default): per
  // caller row x beam, the occupied cell iy*W+ix each ray stopped in (-1:
  // max range / grid exit) for the post-step scan (store_states rows) and the
  // scan behind the returned states rows, and that scan's noisy clipped range
  // in cm (SimBatch.last_scan, core.py:97, 237-241).  Only the kRec kernel
  // instantiation writes them.
  int32_t* hit_store;
  int32_t* hit_state;
  double* scan_state;
};

struct ScanArgs {
  int64_t n;
  const int64_t* cta_begin;     // grid + 1 query boundaries
  const int64_t* qoff;          // n_maps + 1 query ranges (device copy)
  const double *x, *y, *h;
  double* ranges;
  int32_t* hit_cell;
};

}  // namespace sp
