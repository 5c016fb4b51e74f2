// sp_capi.cu -- extern "C" implementation of include/sparrow.h.
//
// Host responsibilities: map preprocessing (bit-packing, the per-cell
// free-box table by an exact chessboard distance transform), map-major slot
// ordering, device SoA allocation, launch geometry (one CTA per SM, shared
// memory = one map's tables + the chunk scratch), error codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sp_env.cu"
#include "sp_ops.cu"
#include "sp_learn.cu"
#include "sp_actor.cu"

using namespace sp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SP_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(SP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)

constexpr int kMaxWarps = SP_CTA_THREADS / 32;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int grid_for(int64_t n, int block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, 148 * 16));
}

struct DevDeviceGuard {
  int prev = -1;
  explicit DevDeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevDeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Per-cell free-box table (the march's table): an occupied cell stores 0x80
// (negative as a signed byte); a free cell stores r = (chessboard distance to
// the nearest occupied or out-of-grid cell) - 1, clamped to 127: the
// (2r+1) x (2r+1) cells centred on it are all free.  Exact two-pass
// chessboard distance transform.
void build_cell_table(const uint8_t* occ, int H, int W, uint8_t* out) {
  std::vector<int> dist((size_t)H * W);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const int border = std::min(std::min(x + 1, y + 1), std::min(W - x, H - y));
      dist[(size_t)y * W + x] = occ[(size_t)y * W + x] ? 0 : border;
    }
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int& d = dist[(size_t)y * W + x];
      if (x > 0) d = std::min(d, dist[(size_t)y * W + x - 1] + 1);
      if (y > 0) {
        d = std::min(d, dist[(size_t)(y - 1) * W + x] + 1);
        if (x > 0) d = std::min(d, dist[(size_t)(y - 1) * W + x - 1] + 1);
        if (x + 1 < W) d = std::min(d, dist[(size_t)(y - 1) * W + x + 1] + 1);
      }
    }
  for (int y = H - 1; y >= 0; --y)
    for (int x = W - 1; x >= 0; --x) {
      int& d = dist[(size_t)y * W + x];
      if (x + 1 < W) d = std::min(d, dist[(size_t)y * W + x + 1] + 1);
      if (y + 1 < H) {
        d = std::min(d, dist[(size_t)(y + 1) * W + x] + 1);
        if (x + 1 < W) d = std::min(d, dist[(size_t)(y + 1) * W + x + 1] + 1);
        if (x > 0) d = std::min(d, dist[(size_t)(y + 1) * W + x - 1] + 1);
      }
    }
  for (size_t i = 0; i < dist.size(); ++i)
    out[i] = dist[i] == 0 ? (uint8_t)0x80u : (uint8_t)std::min(dist[i] - 1, 127);
}

// every map's border row/column fully occupied (GridMap's invariant,
// gridmap.py:90-95): no march step can then leave the grid
bool all_bordered(const SpMapDesc* maps, int n_maps) {
  for (int m = 0; m < n_maps; ++m) {
    const int H = maps[m].n_rows, W = maps[m].n_cols;
    const uint8_t* o = maps[m].occupancy;
    for (int ix = 0; ix < W; ++ix)
      if (!o[ix] || !o[(size_t)(H - 1) * W + ix]) return false;
    for (int iy = 0; iy < H; ++iy)
      if (!o[(size_t)iy * W] || !o[(size_t)iy * W + W - 1]) return false;
  }
  return true;
}

}  // namespace

struct SpEnv {
  int device = 0;
  EnvDev d{};
  int64_t n = 0;
  int R = 0, D = 0, n_maps = 0;
  bool auto_reset = true;
  uint64_t step_index = 0;
  std::vector<int64_t> env_of_slot, slot_of_env, map_off;
  std::vector<void*> allocs;
  int grid = 0, threads = 0;
  size_t smem = 0;
  int n_sm = 0, smem_optin = 0, smem_per_sm = 0;
  int32_t* h_err = nullptr;  // pinned
  int64_t* h_scan = nullptr;  // pinned staging for scan offsets (n_maps + 1 + n_sm + 1)
  int64_t* d_scan = nullptr;
  cudaEvent_t scan_copied = nullptr;
  uint8_t* d_host_stage = nullptr;  // sp_env_step_host: actions | output block (device)
  // sp_env_set_recording: hit cells / noisy ranges of every launch (null = off)
  int32_t* rec_hit_store = nullptr;
  int32_t* rec_hit_state = nullptr;
  double* rec_scan_state = nullptr;
  unsigned long long* d_count = nullptr;  // sp_env_first_pending scratch
  // one-shot re-plan (replan_by_cost): the CTA cycles of the third step launch,
  // read back asynchronously, give each map's cost; CTAs are then allocated
  // to maps by cost instead of by lane count
  int replan_state = 0;  // 0 waiting, 1 cycles in flight, 2 done (or off)
  uint64_t step_launches = 0;
  uint32_t* cyc_host = nullptr;  // pinned, grid
  cudaEvent_t cyc_ready = nullptr;
  // sp_env_step_host row parts: part p's rows are stepped by a launch with the
  // launch plan of dpart[p] (only its plan fields are used) and copied back
  // while the next part steps
  std::vector<EnvDev> dpart;
  std::vector<int64_t> part_rows;  // parts + 1 row cuts
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t part_done[8] = {};
  cudaEvent_t acts_rest = nullptr;  // the actions of parts 1.. landed (copy stream)
  std::mutex mu;

  template <class T>
  int alloc(T** p, size_t count, int fill_byte = 0) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count * sizeof(T), 16));
    if (e != cudaSuccess) return fail(SP_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    cudaMemset(q, fill_byte, std::max<size_t>(count * sizeof(T), 16));
    allocs.push_back(q);
    *p = (T*)q;
    return SP_OK;
  }
  ~SpEnv() {
    for (void* p : allocs) cudaFree(p);
    if (h_err) cudaFreeHost(h_err);
    if (cyc_host) cudaFreeHost(cyc_host);
    if (cyc_ready) cudaEventDestroy(cyc_ready);
    for (cudaEvent_t e : part_done)
      if (e) cudaEventDestroy(e);
    if (acts_rest) cudaEventDestroy(acts_rest);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (h_scan) cudaFreeHost(h_scan);
    if (scan_copied) cudaEventDestroy(scan_copied);
  }
};

struct SpReplay {
  int device = 0;
  int64_t cap = 0, cursor = 0, size = 0;
  int32_t dim = 0;
  float *s = nullptr, *r = nullptr, *s2 = nullptr;
  int64_t* a = nullptr;
  uint8_t* dn = nullptr;
  int64_t* d_size = nullptr;  // device copy of `size` (written by the append kernel)
  std::mutex mu;
  ~SpReplay() {
    cudaFree(s); cudaFree(r); cudaFree(s2); cudaFree(a); cudaFree(dn); cudaFree(d_size);
  }
};

// Launch geometry shared by the step and scan kernels.
struct Plan {
  int grid = 1, threads = 768, chunk_cap = 1, slot_cap = 33, smem_maps = 1;
  size_t smem = 0;
  std::vector<int64_t> cta_begin;  // grid + 1
};

// CTA slot ranges: every CTA stays inside one map when there are at most as
// many non-empty maps as CTAs (CTAs per map proportional to its lanes -- or
// to the map's measured cost `w` when given -- largest remainder); otherwise
// equal contiguous splits.
static std::vector<int64_t> cta_ranges(const std::vector<int64_t>& off, int G,
                                       const std::vector<double>* w = nullptr) {
  const int M = (int)off.size() - 1;
  const int64_t N = off[M] - off[0];
  std::vector<int64_t> b;
  int nonempty = 0;
  for (int m = 0; m < M; ++m) nonempty += off[m + 1] > off[m];
  if (N <= 0) return {off[0], off[0]};
  if (nonempty > G || nonempty == 0) {
    for (int c = 0; c <= G; ++c) b.push_back(off[0] + N * c / G);
    return b;
  }
  // a map's load: its lanes, or its measured cost (zero for an empty map)
  std::vector<double> ld(M);
  double L = 0.0;
  for (int m = 0; m < M; ++m) {
    const int64_t nm = off[m + 1] - off[m];
    ld[m] = nm == 0 ? 0.0 : (w ? std::max((*w)[m], 1e-9) : (double)nm);
    L += ld[m];
  }
  std::vector<int> g(M, 0);
  int used = 0;
  for (int m = 0; m < M; ++m) {
    const int64_t nm = off[m + 1] - off[m];
    if (nm == 0) continue;
    g[m] = std::max<int>(1, (int)(ld[m] * G / L));
    used += g[m];
  }
  while (used > G) {  // too many after the min-1 rule: trim the best-served map
    int best = -1;
    for (int m = 0; m < M; ++m)
      if (g[m] > 1 && (best < 0 || ld[m] * g[best] < ld[best] * g[m])) best = m;
    if (best < 0) break;
    --g[best];
    --used;
  }
  while (used < G) {  // hand spare CTAs to the map with the most load per CTA
    int best = -1;
    for (int m = 0; m < M; ++m)
      if (g[m] > 0 && (best < 0 || ld[m] * g[best] > ld[best] * g[m])) best = m;
    const int64_t nm = off[best + 1] - off[best];
    if (g[best] >= nm) break;
    ++g[best];
    ++used;
  }
  b.push_back(off[0]);
  for (int m = 0; m < M; ++m) {
    const int64_t nm = off[m + 1] - off[m];
    for (int c = 1; c <= g[m]; ++c) b.push_back(off[m] + nm * c / g[m]);
  }
  return b;
}

// shared-memory bytes of a chunk with `cap` envs (layout of chunk_smem)
static int extra_slots(int cap) { return std::max(32, cap / 8); }
static size_t chunk_bytes(int cap, int D, int R) {
  // layout of chunk_smem (chunk_offsets): 109 B per scan slot, 30 B per env,
  // control words
  (void)R;
  (void)D;
  uint32_t o[sp::CF_N];
  sp::chunk_offsets(0, cap, cap + extra_slots(cap), o);
  return (size_t)o[sp::CF_END] + 16;
}

static Plan plan_launch(SpEnv* env, const std::vector<int64_t>& off, bool staging = true) {
  const EnvDev& d = env->d;
  const int D = staging ? d.D : 0;  // the scan kernel stages nothing
  Plan p;
#ifdef SP_SCAN_THREADS
  const int max_threads = staging ? kMaxWarps * 32 : SP_SCAN_THREADS;
#else
  const int max_threads = kMaxWarps * 32;
#endif
  const int64_t lanes = off.back() - off.front();
  const size_t fixed = align_up((size_t)d.R * 16, 128) + 128;
  // per-CTA budget: SP_CTAS_PER_SM CTAs share the SM's shared memory (plus
  // 1 KB per CTA reserved by the driver)
  const size_t sm_total = (size_t)env->smem_per_sm;
  const size_t budget = std::min((size_t)env->smem_optin,
                                 sm_total / SP_CTAS_PER_SM) - 1024
#ifdef SP_TIMING
                        - 1536  // the stamps' static shared memory
#endif
      ;
  size_t map_bytes = align_up(d.map_bytes, 128);
  p.threads = max_threads;
  if (map_bytes + fixed + chunk_bytes(128, D, d.R) + 128 > budget) {
    p.smem_maps = 0;  // map does not fit next to a useful chunk: read tables via L1/L2
    map_bytes = 0;
  }
  const size_t room = budget - fixed - map_bytes - 128;
  int cap = p.threads;
  if (const char* mc = getenv("SPARROW_MAX_CHUNK")) cap = std::max(16, std::min(cap, atoi(mc)));
  while (cap > 1 && chunk_bytes(cap, D, d.R) > room) cap -= 16;
  p.chunk_cap = std::max(1, cap);
  p.slot_cap = p.chunk_cap + extra_slots(p.chunk_cap);
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)env->n_sm * SP_CTAS_PER_SM,
                                                         (lanes + 15) / 16));
  p.cta_begin = cta_ranges(off, p.grid);
  p.grid = (int)p.cta_begin.size() - 1;
  p.smem = map_bytes + fixed + align_up(chunk_bytes(p.chunk_cap, D, d.R), 128);
  return p;
}

static void apply_plan(const Plan& p, EnvDev& d) {
  const size_t map_region = p.smem_maps ? align_up(d.map_bytes, 128) : 0;
  d.off_beam = (uint32_t)map_region;
  d.off_bar = (uint32_t)(map_region + align_up((size_t)d.R * 16, 128));
  d.off_chunk = d.off_bar + 128;
  d.chunk_cap = p.chunk_cap;
  d.slot_cap = p.slot_cap;
  chunk_offsets(d.off_chunk, p.chunk_cap, p.slot_cap, d.co);
  d.smem_maps = p.smem_maps;
}

template <class T>
static int d2h_slots(SpEnv* env, const T* dev, std::vector<T>& host, cudaStream_t st) {
  host.resize(env->n);
  SP_CUDA(cudaMemcpyAsync(host.data(), dev, sizeof(T) * env->n, cudaMemcpyDeviceToHost, st));
  return SP_OK;
}

extern "C" {

const char* sp_last_error(void) { return g_err.c_str(); }
int sp_version(void) { return 1; }

int sp_device_info(int device, int* n_sm, int* smem_optin, int* major, int* minor) {
  cudaDeviceProp p;
  SP_CUDA(cudaGetDeviceProperties(&p, device));
  if (n_sm) *n_sm = p.multiProcessorCount;
  if (smem_optin) *smem_optin = (int)p.sharedMemPerBlockOptin;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  return SP_OK;
}

int sp_env_create(const SpConfig* cfg, const SpMapDesc* maps, int32_t n_maps, int64_t n_envs,
                  const int32_t* map_index, const SpRanges* ranges, int64_t n_ranges,
                  int64_t env_id_offset, int device, SpEnv** out) {
  if (!cfg || !maps || !out || n_maps < 1) return fail(SP_EINVAL, "null argument");
  if (n_envs < 1) return fail(SP_EINVAL, "need at least one copy");  // vecenv.py:66-67
  if (cfg->n_beams < 1) return fail(SP_EINVAL, "n_beams must be >= 1");
  if (!(cfg->max_range_cm > 0.0) || !(cfg->robot_radius_cm >= 0.0) || cfg->spawn_attempts < 1 ||
      cfg->timeout_steps < 1)
    return fail(SP_EINVAL, "config: max range > 0, radius >= 0, spawn attempts >= 1, timeout >= 1");
  if (!cfg->beam_offsets) return fail(SP_EINVAL, "config: beam offsets missing");
  if (cfg->n_actions < 1 || cfg->n_actions > SP_MAX_ACTIONS)
    return fail(SP_EINVAL, "action table must have 1..15 entries");
  if (n_ranges != 1 && n_ranges != n_envs)
    return fail(SP_EINVAL, "need one DiversityRanges per lane");  // core.py:56-57
  const int H = maps[0].n_rows, W = maps[0].n_cols;
  const double cell = maps[0].cell_cm;
  if (!(cell > 0.0)) return fail(SP_EINVAL, "cell size must be positive");
  for (int m = 0; m < n_maps; ++m)
    if (maps[m].n_rows != H || maps[m].n_cols != W || maps[m].cell_cm != cell)
      return fail(SP_EMAP, "all maps in one batch must share grid shape and cell size");
  if (H < 1 || W < 1 || H > (1 << 15) || W > (1 << 15)) return fail(SP_EINVAL, "bad grid shape");
  for (int64_t i = 0; map_index && i < n_envs; ++i)
    if (map_index[i] < 0 || map_index[i] >= n_maps)
      return fail(SP_EINVAL, "map_index out of range");  // core.py:58-59
  for (int64_t r = 0; r < n_ranges; ++r)
    if (ranges[r].delay[0] < 0 || ranges[r].delay[1] > SP_MAX_DELAY ||
        ranges[r].delay[0] > ranges[r].delay[1])
      return fail(SP_EINVAL, "control delay range must lie in [0, 64]");
  // GridMap's invariant (gridmap.py:90-95): the marcher relies on it (no step
  // can leave the grid); the op-level seam sp_cast_rays takes any grid
  if (!all_bordered(maps, n_maps)) return fail(SP_EMAP, "border cells must all be occupied");

  DevDeviceGuard guard(device);
  SpEnv* env = new SpEnv();
  env->device = device;
  env->n = n_envs;
  env->R = cfg->n_beams;
  env->D = 5 + cfg->n_beams;
  env->n_maps = n_maps;
  env->auto_reset = cfg->auto_reset != 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    delete env;
    return fail(SP_ECUDA, "cudaGetDeviceProperties failed");
  }
  env->n_sm = prop.multiProcessorCount;
  env->smem_optin = (int)prop.sharedMemPerBlockOptin;
  env->smem_per_sm = (int)prop.sharedMemPerMultiprocessor;

  EnvDev& d = env->d;
  d.n = n_envs;
  d.R = env->R;
  d.D = env->D;
  d.H = H;
  d.W = W;
  d.Hb = H;  // the march table is per cell (build_cell_table)
  d.Wb = W;
  d.WW = (W + 31) / 32;
  d.n_maps = n_maps;
  d.cell = cell;
  d.inv_cell = 1.0 / cell;
  d.max_range = cfg->max_range_cm;
  d.radius = cfg->robot_radius_cm;
  d.proximity = cfg->proximity_cm;
  d.timeout = cfg->timeout_steps;
  d.spawn_attempts = cfg->spawn_attempts;
  d.auto_reset = cfg->auto_reset ? 1 : 0;
  d.n_actions = cfg->n_actions;
  {
    const int K = (int)std::ceil(cfg->robot_radius_cm / cell);
    // a cell box of radius >= K around the disc's centre cell covers its cell
    // bbox.  disc_hits finds the centre cell as floor(x * inv_cell): exact
    // when the cell size is a power of two, else it may land one cell off
    // next to a cell edge, which one more ring of free cells absorbs
    int e2 = 0;
    const bool pow2 = std::frexp(cell, &e2) == 0.5;
    d.need_k = K + (pow2 ? 0 : 1);
  }
  for (int c = 0; c <= SP_MAX_ACTIONS; ++c) {
    d.action_v[c] = c < cfg->n_actions ? cfg->action_table[2 * c] : 0.0;
    d.action_w[c] = c < cfg->n_actions ? cfg->action_table[2 * c + 1] : 0.0;
  }
  d.action_v[SP_MAX_ACTIONS] = 0.0;  // the (0, 0) delay filler (core.py:156)
  d.action_w[SP_MAX_ACTIONS] = 0.0;
  d.blk_bytes = (uint32_t)align_up((size_t)d.Hb * d.Wb, 16);
  d.bits_bytes = (uint32_t)align_up((size_t)H * d.WW * 4, 16);
  d.map_bytes = d.blk_bytes + d.bits_bytes;
  d.env_id_offset = env_id_offset;
  // default assignment (map = (env_id_offset + row) % n_maps, also when the
  // caller passes it explicitly, as VecEnv does): rows follow from slots
  // arithmetically, so the kernel never loads env_of_slot
  bool affine = true;
  if (map_index) {
    const int64_t om = ((env_id_offset % n_maps) + n_maps) % n_maps;
    for (int64_t i = 0; i < n_envs && affine; ++i)
      affine = map_index[i] == (int32_t)((om + i) % n_maps);
  }
  d.row_affine = affine ? 1 : 0;
  d.off_mod = (int32_t)(((env_id_offset % n_maps) + n_maps) % n_maps);

  // slot order: stable sort by map (map-major)
  std::vector<int32_t> midx(n_envs);
  for (int64_t i = 0; i < n_envs; ++i)
    midx[i] = map_index ? map_index[i] : (int32_t)((env_id_offset + i) % n_maps);
  env->map_off.assign(n_maps + 1, 0);
  for (int64_t i = 0; i < n_envs; ++i) env->map_off[midx[i] + 1]++;
  for (int m = 0; m < n_maps; ++m) env->map_off[m + 1] += env->map_off[m];
  env->env_of_slot.resize(n_envs);
  env->slot_of_env.resize(n_envs);
  {
    std::vector<int64_t> fillp(env->map_off.begin(), env->map_off.end() - 1);
    for (int64_t i = 0; i < n_envs; ++i) {
      int64_t s = fillp[midx[i]]++;
      env->env_of_slot[s] = i;
      env->slot_of_env[i] = s;
    }
  }

  // map tables + constants
  std::vector<uint8_t> host_maps((size_t)n_maps * d.map_bytes, 0);
  std::vector<MapConst> mconst(n_maps);
  for (int m = 0; m < n_maps; ++m) {
    uint8_t* base = host_maps.data() + (size_t)m * d.map_bytes;
    build_cell_table(maps[m].occupancy, H, W, base);
    uint32_t* bits = (uint32_t*)(base + d.blk_bytes);
    for (int iy = 0; iy < H; ++iy)
      for (int ix = 0; ix < W; ++ix)
        if (maps[m].occupancy[(size_t)iy * W + ix]) bits[(size_t)iy * d.WW + (ix >> 5)] |= 1u << (ix & 31);
    mconst[m].goal_x = maps[m].goal_x;
    mconst[m].goal_y = maps[m].goal_y;
    mconst[m].goal_r = maps[m].goal_radius;
    mconst[m].plan_dist = maps[m].planning_dist;
    mconst[m].inv_plan = 1.0 / maps[m].planning_dist;
    for (int k = 0; k < 4; ++k) mconst[m].spawn[k] = maps[m].spawn[k];
  }
  std::vector<double2> beam(env->R);
  for (int j = 0; j < env->R; ++j) beam[j] = make_double2(std::cos(cfg->beam_offsets[j]), std::sin(cfg->beam_offsets[j]));
  std::vector<double> rng_rows((size_t)(n_ranges == 1 ? 1 : n_envs) * 12);
  for (int64_t s = 0; s < (n_ranges == 1 ? 1 : n_envs); ++s) {
    const SpRanges& r = ranges[n_ranges == 1 ? 0 : env->env_of_slot[s]];
    double* o = rng_rows.data() + 12 * s;
    o[0] = r.k[0]; o[1] = r.k[1]; o[2] = r.dt[0]; o[3] = r.dt[1];
    o[4] = r.delay[0]; o[5] = r.delay[1]; o[6] = r.vmax_linear[0]; o[7] = r.vmax_linear[1];
    o[8] = r.vmax_angular[0]; o[9] = r.vmax_angular[1]; o[10] = r.noise_std[0]; o[11] = r.noise_std[1];
  }
  d.ranges_shared = n_ranges == 1;

  int rc = SP_OK;
  uint8_t* dmaps; MapConst* dmc; int64_t* dmoff; double2* dbeam; double* drng; int64_t* deos;
#define TRY(x) do { rc = (x); if (rc) { delete env; return rc; } } while (0)
  TRY(env->alloc(&dmaps, host_maps.size()));
  TRY(env->alloc(&dmc, n_maps));
  TRY(env->alloc(&dmoff, n_maps + 1));
  TRY(env->alloc(&dbeam, env->R));
  TRY(env->alloc(&drng, rng_rows.size()));
  TRY(env->alloc(&deos, n_envs));
  const size_t n = (size_t)n_envs;
  double** f64s[] = {&d.x, &d.y, &d.h, &d.vl, &d.va, &d.ret, &d.sx, &d.sy, &d.c0, &d.s0,
                     &d.pk, &d.pdt, &d.pvl, &d.pva, &d.psig, &d.return_sum, &d.first_ret};
  for (double** p : f64s) TRY(env->alloc(p, n));
  TRY(env->alloc(&d.hist, 4 * n, 0xff));
  TRY(env->alloc(&d.ctr, n));
  TRY(env->alloc(&d.step, n));
  TRY(env->alloc(&d.delay, n));
  TRY(env->alloc(&d.needs_reset, n, 1));
  TRY(env->alloc(&d.qhist, n, 0x80));  // no history yet: every group ranks longest
  TRY(env->alloc(&d.episodes, n));
  TRY(env->alloc(&d.arrivals, n));
  TRY(env->alloc(&d.first_event, n, 0xff));
  TRY(env->alloc(&d.first_steps, n));
  d.rec_cap = (uint64_t)align_up(n + 256, 256);
  TRY(env->alloc(&d.rec_ret, d.rec_cap));
  TRY(env->alloc(&d.rec_key, d.rec_cap));
  TRY(env->alloc(&d.rec_count, 1));
  TRY(env->alloc(&d.err, 4));
#undef TRY
  if (cudaMallocHost(&env->h_err, 16) != cudaSuccess ||
      cudaMallocHost(&env->h_scan, 8 * (size_t)(n_maps + env->n_sm * SP_CTAS_PER_SM + 2)) != cudaSuccess ||
      env->alloc(&env->d_scan, (size_t)(n_maps + env->n_sm * SP_CTAS_PER_SM + 2)) != SP_OK ||
      cudaEventCreateWithFlags(&env->scan_copied, cudaEventDisableTiming) != cudaSuccess) {
    delete env;
    return fail(SP_ENOMEM, "pinned alloc");
  }
  cudaMemcpy(dmaps, host_maps.data(), host_maps.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dmc, mconst.data(), sizeof(MapConst) * n_maps, cudaMemcpyHostToDevice);
  cudaMemcpy(dmoff, env->map_off.data(), sizeof(int64_t) * (n_maps + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dbeam, beam.data(), sizeof(double2) * env->R, cudaMemcpyHostToDevice);
  cudaMemcpy(drng, rng_rows.data(), sizeof(double) * rng_rows.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(deos, env->env_of_slot.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice);
  d.maps = dmaps;
  d.mconst = dmc;
  d.map_off = dmoff;
  d.beam_cs = dbeam;
  d.ranges = drng;
  d.env_of_slot = deos;

  {
    const int R = env->R;
    int gs = 0;  // beams per dispatch group: the power of two >= R / 8
    while ((8 << gs) < R) ++gs;
    if (const char* g = std::getenv("SPARROW_GSHIFT"))  // experiments: larger groups
      gs = std::max(gs, std::min(10, std::atoi(g)));
    d.gshift = gs;
    d.n_groups = (R + (1 << gs) - 1) >> gs;
    d.d_magic = (((uint64_t)1 << 40) + (uint64_t)env->D - 1) / (uint64_t)env->D;
    d.nb = (R + 3) / 4;
    d.nb_shift = (d.nb & (d.nb - 1)) == 0 ? __builtin_ctz((unsigned)d.nb) : -1;
    d.inv_max_range = 1.0 / cfg->max_range_cm;
    const char* rm = std::getenv("SPARROW_REFILL_MIN");
    d.refill_min = rm ? std::max(1, std::min(64, std::atoi(rm))) : 40;
    const char* pn = std::getenv("SPARROW_PRENOISE");
    d.prenoise = pn ? std::max(0, std::min(64, std::atoi(pn))) : 24;
    const char* lr = std::getenv("SPARROW_LATE_RESETS");  // tests / A/B: 0 = inline resets
    d.late_resets = lr && lr[0] == '0' ? 0 : 1;
  }
  Plan plan = plan_launch(env, env->map_off);
  apply_plan(plan, d);
  int64_t* dcta = nullptr;
  {
    int rc2 = env->alloc(&dcta, plan.cta_begin.size());
    if (!rc2) rc2 = env->alloc(&d.cta_cyc, plan.cta_begin.size());
    if (rc2) { delete env; return rc2; }
    cudaMemcpy(dcta, plan.cta_begin.data(), 8 * plan.cta_begin.size(), cudaMemcpyHostToDevice);
  }
  d.cta_begin = dcta;
  d.plan_n = 0;
  if (plan.grid <= SP_PLAN_MAX && n_envs < (int64_t)1 << 31) {  // the plan rides in the params
    d.plan_n = plan.grid;
    for (int b = 0; b <= plan.grid; ++b) d.plan_begin[b] = (int32_t)plan.cta_begin[b];
    for (int b = 0; b < plan.grid; ++b) d.plan_end[b] = (int32_t)plan.cta_begin[b + 1];
    for (int b = 0; b < plan.grid; ++b) {
      int m = 0;
      while (env->map_off[m + 1] <= plan.cta_begin[b] && m + 1 < n_maps) ++m;
      d.plan_map[b] = (int16_t)m;
      d.plan_mstart[b] = (int32_t)env->map_off[m];
      d.plan_mend[b] = (int32_t)env->map_off[m + 1];
    }
    if (n_maps > 32767) d.plan_n = 0;
  }
  {
    const char* rpe = std::getenv("SPARROW_REPLAN");  // 0: keep the lane-count plan
    env->replan_state = 2;
    if (d.plan_n > 0 && !(rpe && rpe[0] == '0') &&
        cudaMallocHost(&env->cyc_host, 4 * (size_t)d.plan_n) == cudaSuccess &&
        cudaEventCreateWithFlags(&env->cyc_ready, cudaEventDisableTiming) == cudaSuccess)
      env->replan_state = 0;
  }
  env->grid = plan.grid;
  env->threads = plan.threads;
  env->smem = plan.smem;
  // sp_env_step_host row parts (default from 16,384 envs: two, a quarter of the
  // rows then the rest; SPARROW_HOST_PARTS sets an even split into that many,
  // 1 = off; SPARROW_HOST_PART_W="w0,w1,..." weights them): for the default
  // map assignment a row range holds, per map, one contiguous slot range, so
  // each part gets its own launch plan.  A launch costs ~40 us whatever its
  // size (cfg2's 4,096 envs step in 40 us), so the first part is small only
  // to start the copies early, and few parts pay: the copies (~95 us per
  // 16,384 rows) are the floor.  e2e per step at cfg3: four even parts
  // 0.488 / 0.497 ms, three (1:2:5) 0.478 / 0.478, two (1:3) 0.473 / 0.477.
  {
    const char* hp = std::getenv("SPARROW_HOST_PARTS");
    if (hp && !*hp) hp = nullptr;  // set but empty: the default
    const char* pw = std::getenv("SPARROW_HOST_PART_W");
    std::string wspec = pw ? pw : (hp ? "" : "1,3");
    int parts = hp ? std::max(1, std::min(8, std::atoi(hp))) : (n_envs >= 16384 ? 2 : 1);
    if (!(d.plan_n > 0 && d.row_affine && d.smem_maps)) parts = 1;
    if (parts > 1) {
      const int M = n_maps;
      std::vector<int64_t> rows(parts + 1);
      for (int p = 0; p <= parts; ++p) rows[p] = n_envs * p / parts;
      if (!wspec.empty()) {  // part weights
        std::vector<double> w;
        for (const char* q = wspec.c_str(); *q;) {
          w.push_back(std::atof(q));
          while (*q && *q != ',') ++q;
          if (*q == ',') ++q;
        }
        if ((int)w.size() == parts) {
          double tot = 0, acc = 0;
          for (double x : w) tot += x;
          for (int p = 0; p < parts; ++p) {
            acc += w[p];
            rows[p + 1] = p + 1 == parts ? n_envs : (int64_t)(n_envs * acc / tot);
          }
        }
      }
      std::vector<EnvDev> dps;
      bool ok = true;
      for (int p = 0; p < parts && ok; ++p) {
        // per map m: slots [lo[m], hi[m]) have rows in [rows[p], rows[p + 1])
        std::vector<int64_t> lo(M), hi(M), voff(M + 1, 0);
        for (int m = 0; m < M; ++m) {
          const int64_t i0 = m >= d.off_mod ? m - d.off_mod : m - d.off_mod + M;
          const int64_t nm = env->map_off[m + 1] - env->map_off[m];
          auto first_j = [&](int64_t r) {  // first j with i0 + j * M >= r
            return std::min(nm, std::max<int64_t>(0, (r - i0 + M - 1) / M));
          };
          lo[m] = env->map_off[m] + first_j(rows[p]);
          hi[m] = env->map_off[m] + first_j(rows[p + 1]);
          voff[m + 1] = voff[m] + (hi[m] - lo[m]);
        }
        const std::vector<int64_t> vc = cta_ranges(voff, plan.grid);
        const int G = (int)vc.size() - 1;
        EnvDev dp = d;
        dp.plan_n = G;
        for (int b = 0; b < G && ok; ++b) {
          int m = 0;
          while (m + 1 < M && voff[m + 1] <= vc[b]) ++m;
          if (vc[b + 1] > voff[m + 1]) ok = false;  // a CTA would span two maps
          dp.plan_begin[b] = (int32_t)(lo[m] + (vc[b] - voff[m]));
          dp.plan_end[b] = (int32_t)(lo[m] + (vc[b + 1] - voff[m]));
          if (dp.plan_end[b] - dp.plan_begin[b] > d.chunk_cap) ok = false;
          dp.plan_map[b] = (int16_t)m;
          dp.plan_mstart[b] = (int32_t)env->map_off[m];
          dp.plan_mend[b] = (int32_t)env->map_off[m + 1];
        }
        dps.push_back(dp);
      }
      if (ok && cudaStreamCreateWithFlags(&env->copy_stream, cudaStreamNonBlocking) == cudaSuccess) {
        for (int p = 0; p < parts && ok; ++p)
          ok = cudaEventCreateWithFlags(&env->part_done[p], cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&env->acts_rest, cudaEventDisableTiming) == cudaSuccess;
        if (ok) {
          env->dpart = dps;
          env->part_rows = rows;
        }
      }
    }
  }
  const void* kernels_[] = {(const void*)env_step_kernel<true, false>,
                            (const void*)env_step_kernel<false, false>,
                            (const void*)env_step_kernel<true, true>,
                            (const void*)env_step_kernel<false, true>,
                            (const void*)env_scan_kernel<true>, (const void*)env_scan_kernel<false>};
  cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
  for (const void* k : kernels_) {
    cudaFuncAttributes fa;  // static shared memory (debug stamp builds) counts against the opt-in
    const size_t stat = cudaFuncGetAttributes(&fa, k) == cudaSuccess ? fa.sharedSizeBytes : 0;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         env->smem_optin - (int)stat);
    if (e != cudaSuccess) e1 = e;
  }
  cudaError_t e3 = cudaDeviceSynchronize();
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
    delete env;
    return fail(SP_ECUDA, std::string("env setup: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3)));
  }
  *out = env;
  return SP_OK;
}

int sp_env_destroy(SpEnv* env) {
  if (!env) return SP_OK;
  DevDeviceGuard guard(env->device);
  cudaDeviceSynchronize();
  delete env;
  return SP_OK;
}

// Allocate the step's CTAs to maps by measured cost (one CTA's time = a fixed
// part, ~40 % of the median, + its envs' variable cost): the maps' costs
// differ by +-5 % and the pattern persists from step to step, so the extra
// CTAs go to the costliest maps.  Cuts inside a map stay equal-count; results
// do not depend on the plan (every lane's computation is its own).
static void replan_by_cost(SpEnv* env) {
  EnvDev& d = env->d;
  const int G = d.plan_n, M = env->n_maps;
  std::vector<double> y(env->cyc_host, env->cyc_host + G), ys = y;
  std::nth_element(ys.begin(), ys.begin() + G / 2, ys.end());
  const double F = 0.4 * ys[G / 2];
  std::vector<double> w(M, 0.0);
  for (int b = 0; b < G; ++b) w[d.plan_map[b]] += std::max(y[b] - F, 0.05 * y[b]);
  // per map cost per lane (normalised by its lanes: the maps' lane counts may
  // differ), then only the spare CTAs move: every map keeps the count the
  // lane plan gives the smallest-served map, the G % M extra ones go to the
  // costliest maps (one step's estimate is noisy, so never fewer CTAs than a
  // lane-count plan would give)
  std::vector<int> g(M, 0);
  for (int b = 0; b < G; ++b) ++g[d.plan_map[b]];
  int base = G;
  for (int m = 0; m < M; ++m)
    if (env->map_off[m + 1] > env->map_off[m]) base = std::min(base, g[m]);
  int used = 0;
  for (int m = 0; m < M; ++m) {
    g[m] = env->map_off[m + 1] > env->map_off[m] ? base : 0;
    used += g[m];
  }
  while (used < G) {  // the spare CTAs, one at a time, to the highest cost per CTA
    int best = -1;
    for (int m = 0; m < M; ++m)
      if (g[m] > 0 && (best < 0 || w[m] * g[best] > w[best] * g[m])) best = m;
    if (best < 0) return;
    ++g[best];
    ++used;
  }
  std::vector<int64_t> cuts{env->map_off[0]};
  for (int m = 0; m < M; ++m) {
    const int64_t nm = env->map_off[m + 1] - env->map_off[m];
    for (int c = 1; c <= g[m]; ++c) cuts.push_back(env->map_off[m] + nm * c / g[m]);
  }
  if ((int)cuts.size() != G + 1) return;
  for (int b = 0; b < G; ++b) {
    if (cuts[b + 1] - cuts[b] > d.chunk_cap) return;  // keep the lane-count plan
    int m = 0;
    while (env->map_off[m + 1] <= cuts[b] && m + 1 < M) ++m;
    if (cuts[b + 1] > env->map_off[m + 1]) return;
  }
  for (int b = 0; b <= G; ++b) d.plan_begin[b] = (int32_t)cuts[b];
  for (int b = 0; b < G; ++b) {
    int m = 0;
    while (env->map_off[m + 1] <= cuts[b] && m + 1 < M) ++m;
    d.plan_end[b] = (int32_t)cuts[b + 1];
    d.plan_map[b] = (int16_t)m;
    d.plan_mstart[b] = (int32_t)env->map_off[m];
    d.plan_mend[b] = (int32_t)env->map_off[m + 1];
  }
}

static int launch_env(SpEnv* env, StepArgs a, cudaStream_t st, const EnvDev* dp = nullptr) {
  // the one-shot re-plan: step launches of the main plan outside graph capture
  bool rp = !dp && env->replan_state < 2 && a.mode == MODE_STEP;
  if (rp) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    rp = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
  }
  if (rp && env->replan_state == 1 && cudaEventQuery(env->cyc_ready) == cudaSuccess) {
    replan_by_cost(env);
    env->replan_state = 2;
  }
  const EnvDev& d = dp ? *dp : env->d;
  const int grid = dp ? dp->plan_n : env->grid;
  a.hit_store = env->rec_hit_store;
  a.hit_state = env->rec_hit_state;
  a.scan_state = env->rec_scan_state;
  const bool rec = a.hit_store || a.hit_state || a.scan_state;
  if (d.smem_maps) {
    if (rec)
      env_step_kernel<true, true><<<grid, env->threads, env->smem, st>>>(d, a);
    else
      env_step_kernel<true, false><<<grid, env->threads, env->smem, st>>>(d, a);
  } else {
    if (rec)
      env_step_kernel<false, true><<<grid, env->threads, env->smem, st>>>(d, a);
    else
      env_step_kernel<false, false><<<grid, env->threads, env->smem, st>>>(d, a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SP_ECUDA, std::string("env_step_kernel: ") + cudaGetErrorString(e));
  if (rp && env->replan_state == 0 && ++env->step_launches == 3) {
    SP_CUDA(cudaMemcpyAsync(env->cyc_host, env->d.cta_cyc, 4 * (size_t)env->d.plan_n,
                            cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaEventRecord(env->cyc_ready, st));
    env->replan_state = 1;
  }
  return SP_OK;
}

int sp_env_set_recording(SpEnv* env, int32_t* hit_store, int32_t* hit_state,
                         double* scan_state) {
  if (!env) return fail(SP_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(env->mu);
  env->rec_hit_store = hit_store;
  env->rec_hit_state = hit_state;
  env->rec_scan_state = scan_state;
  return SP_OK;
}

int sp_env_reset_all(SpEnv* env, uint64_t seed, float* states, void* stream) {
  if (!env || !states) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  cudaStream_t st = (cudaStream_t)stream;
  env->d.seed = seed;
  // step_index keeps increasing across reset_all: the recent-returns ring is
  // keyed (step_index << 32 | row), and the reference's deque keeps appending
  // in time order across resets (vecenv.py:79, 109)
  SP_CUDA(cudaMemsetAsync(env->d.ctr, 0, sizeof(uint64_t) * env->n, st));
  SP_CUDA(cudaMemsetAsync(env->d.err, 0, 16, st));
  StepArgs a{};
  a.mode = MODE_RESET_ALL;
  a.states = states;
  return launch_env(env, a, st);
}

static int step_locked(SpEnv* env, const int64_t* actions, float* states, float* store_states,
                       double* rewards, uint8_t* dones, uint8_t* truncated, int8_t* events,
                       cudaStream_t stream);

int sp_env_step(SpEnv* env, const int64_t* actions, float* states, float* store_states,
                double* rewards, uint8_t* dones, uint8_t* truncated, int8_t* events,
                void* stream) {
  if (!env || !actions || !states || !store_states || !rewards || !dones || !truncated || !events)
    return fail(SP_EINVAL, "null argument");
  {
    const uintptr_t rb = (uintptr_t)env->n * (uintptr_t)env->D * sizeof(float);
    const uintptr_t s0 = (uintptr_t)states, s1 = (uintptr_t)store_states;
    if (s0 < s1 + rb && s1 < s0 + rb)
      return fail(SP_EINVAL, "states and store_states must not overlap");
  }
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  return step_locked(env, actions, states, store_states, rewards, dones, truncated, events,
                     (cudaStream_t)stream);
}

static int step_locked(SpEnv* env, const int64_t* actions, float* states, float* store_states,
                       double* rewards, uint8_t* dones, uint8_t* truncated, int8_t* events,
                       cudaStream_t stream) {
  StepArgs a{};
  a.mode = MODE_STEP;
  a.step_index = ++env->step_index;
  a.actions = actions;
  a.states = states;
  a.store_states = store_states;
  a.rewards = rewards;
  a.dones = dones;
  a.truncated = truncated;
  a.events = events;
  return launch_env(env, a, stream);
}

int64_t sp_env_host_out_bytes(SpEnv* env) {
  if (!env) return -1;
  return env->n * (8 + 2 * 4 * (int64_t)env->D + 3);
}

// The first action outside [0, n_actions) (core.py:169-170), or -1: one
// branch-free pass (a maximum of the unsigned values), then the index.
static int64_t first_bad_action(const int64_t* a, int64_t n, int64_t n_actions) {
  uint64_t mx = 0;
  for (int64_t i = 0; i < n; ++i) mx = std::max(mx, (uint64_t)a[i]);
  if (mx < (uint64_t)n_actions) return -1;
  for (int64_t i = 0; i < n; ++i)
    if ((uint64_t)a[i] >= (uint64_t)n_actions) return i;
  return -1;
}

int sp_env_step_host(SpEnv* env, const int64_t* h_actions, void* h_out, void* stream) {
  if (!env || !h_actions || !h_out) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);  // one staging block per handle
  const int64_t n = env->n, D = env->D, out_bytes = sp_env_host_out_bytes(env);
  if (!env->d_host_stage) {
    uint8_t* p = nullptr;
    const int rc = env->alloc(&p, (size_t)(8 * n + out_bytes));
    if (rc != SP_OK) return rc;
    env->d_host_stage = p;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* dev_act = env->d_host_stage;
  uint8_t* o = env->d_host_stage + 8 * n;  // output block, 8-byte aligned
  double* rewards = (double*)o;
  float* states = (float*)(o + 8 * n);
  float* store = states + n * D;
  uint8_t* dones = (uint8_t*)(store + n * D);
  const int parts = (int)env->dpart.size();
  // the actions are checked on the host while their copy is in flight, before
  // any launch: an invalid one raises before anything steps, as in the
  // reference (core.py:169-170), and costs no extra PCIe round trip
  auto check_actions = [&]() -> int {
    const int64_t bad = first_bad_action(h_actions, n, env->d.n_actions);
    if (bad < 0) return SP_OK;
    cudaStreamSynchronize(st);
    if (env->copy_stream) cudaStreamSynchronize(env->copy_stream);
    return fail(SP_EACTION, "action index out of range (env " + std::to_string(bad) + ")");
  };
  if (parts < 2) {
    SP_CUDA(cudaMemcpyAsync(dev_act, h_actions, 8 * n, cudaMemcpyHostToDevice, st));
    if (const int rc = check_actions()) return rc;
    const int rc = step_locked(env, (const int64_t*)dev_act, states, store, rewards, dones,
                               dones + n, (int8_t*)(dones + 2 * n), st);
    if (rc != SP_OK) return rc;
    SP_CUDA(cudaMemcpyAsync(h_out, o, out_bytes, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    return SP_OK;
  }
  // the first part's actions on the step stream, the rest beside its launch
  // on the copy stream (idle until the first part's rows are ready)
  {
    const int64_t r1 = env->part_rows[1];
    SP_CUDA(cudaMemcpyAsync(dev_act, h_actions, 8 * r1, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(dev_act + 8 * r1, h_actions + r1, 8 * (n - r1), cudaMemcpyHostToDevice,
                            env->copy_stream));
    SP_CUDA(cudaEventRecord(env->acts_rest, env->copy_stream));
    if (const int rc = check_actions()) return rc;
  }
  // row parts: part p's launch, then its rows' copies on the copy stream
  // while part p + 1 steps (the PCIe read-back is most of a host step)
  StepArgs a{};
  a.mode = MODE_STEP;
  a.step_index = ++env->step_index;  // one step for every part (ring keys)
  a.actions = (const int64_t*)dev_act;
  a.states = states;
  a.store_states = store;
  a.rewards = rewards;
  a.dones = dones;
  a.truncated = dones + n;
  a.events = (int8_t*)(dones + 2 * n);
  uint8_t* h = (uint8_t*)h_out;
#ifdef SP_HOST_TIMING  // debug: timeline of the parts (stderr)
  cudaEvent_t tev[20];
  for (auto& e : tev) cudaEventCreate(&e);
  int ti = 0;
  cudaEventRecord(tev[ti++], st);
#endif
  for (int p = 0; p < parts; ++p) {
    if (p == 1) SP_CUDA(cudaStreamWaitEvent(st, env->acts_rest, 0));
    // the handle's current parameters (seed etc.) with part p's launch plan
    EnvDev dp = env->d;
    const EnvDev& pp = env->dpart[p];
    dp.plan_n = pp.plan_n;
    std::memcpy(dp.plan_begin, pp.plan_begin, sizeof(dp.plan_begin));
    std::memcpy(dp.plan_end, pp.plan_end, sizeof(dp.plan_end));
    std::memcpy(dp.plan_map, pp.plan_map, sizeof(dp.plan_map));
    std::memcpy(dp.plan_mstart, pp.plan_mstart, sizeof(dp.plan_mstart));
    std::memcpy(dp.plan_mend, pp.plan_mend, sizeof(dp.plan_mend));
    const int rc = launch_env(env, a, st, &dp);
    if (rc != SP_OK) return rc;
    SP_CUDA(cudaEventRecord(env->part_done[p], st));
#ifdef SP_HOST_TIMING
    cudaEventRecord(tev[ti++], st);
#endif
    SP_CUDA(cudaStreamWaitEvent(env->copy_stream, env->part_done[p], 0));
    // the part's obs rows (the bulk: 2 x 148 B per row at R = 32) now; the
    // small per-row columns once, after the last part (every copy costs ~3.5 us)
    const int64_t r0 = env->part_rows[p], r1 = env->part_rows[p + 1], k = r1 - r0;
    const size_t row_f = 4 * (size_t)D;
    const size_t so = 8 * (size_t)n + row_f * r0, ro = 8 * (size_t)n + row_f * (n + r0);
    SP_CUDA(cudaMemcpyAsync(h + so, o + so, row_f * k, cudaMemcpyDeviceToHost, env->copy_stream));
    SP_CUDA(cudaMemcpyAsync(h + ro, o + ro, row_f * k, cudaMemcpyDeviceToHost, env->copy_stream));
#ifdef SP_HOST_TIMING
    cudaEventRecord(tev[ti++], env->copy_stream);
#endif
  }
  {
    const size_t row_f = 4 * (size_t)D, tail = 8 * (size_t)n + 2 * row_f * n;
    SP_CUDA(cudaMemcpyAsync(h, o, 8 * (size_t)n, cudaMemcpyDeviceToHost, env->copy_stream));
    SP_CUDA(cudaMemcpyAsync(h + tail, o + tail, 3 * (size_t)n, cudaMemcpyDeviceToHost,
                            env->copy_stream));
  }
#ifdef SP_HOST_TIMING
  cudaEventRecord(tev[ti++], env->copy_stream);
#endif
  SP_CUDA(cudaStreamSynchronize(env->copy_stream));
  SP_CUDA(cudaStreamSynchronize(st));
#ifdef SP_HOST_TIMING
  {
    float ms;
    fprintf(stderr, "parts timeline (us from start):");
    for (int i = 1; i < ti; ++i) {
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      fprintf(stderr, " %.1f", ms * 1e3f);
    }
    fprintf(stderr, "\n");
    for (auto& e : tev) cudaEventDestroy(e);
  }
#endif
  return SP_OK;
}

int sp_env_check(SpEnv* env, void* stream, int64_t* err_env) {
  if (!env) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  SP_CUDA(cudaMemcpyAsync(env->h_err, env->d.err, 8, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  if (err_env) *err_env = env->h_err[1];
  int code = env->h_err[0];
  if (code != SP_OK) {
    cudaMemsetAsync(env->d.err, 0, 16, st);
    cudaStreamSynchronize(st);
    const char* what = code == SP_EACTION ? "action index out of range"
                       : code == SP_EEPISODE ? "a lane finished its episode; reset before stepping"
                       : code == SP_EMAP ? "no collision-free spawn pose found"
                                         : "device error";
    return fail(code, std::string(what) + " (env " + std::to_string(env->h_err[1]) + ")");
  }
  return SP_OK;
}

int sp_env_any_needs_reset(SpEnv* env, void* stream, int* any) {
  if (!env || !any) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::vector<uint8_t> h(env->n);
  cudaStream_t st = (cudaStream_t)stream;
  SP_CUDA(cudaMemcpyAsync(h.data(), env->d.needs_reset, env->n, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  *any = 0;
  for (int64_t s = 0; s < env->n; ++s)
    if (h[s]) { *any = 1; break; }
  return SP_OK;
}

int sp_env_stats_read(SpEnv* env, int64_t* episodes, int64_t* arrivals, double* return_sum,
                      int8_t* first_event, double* first_return, int64_t* first_steps,
                      void* stream) {
  if (!env) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int64_t> e, a;
  std::vector<double> r, fr;
  std::vector<int8_t> fe;
  std::vector<int32_t> fs;
  int rc;
  if ((rc = d2h_slots(env, env->d.episodes, e, st)) || (rc = d2h_slots(env, env->d.arrivals, a, st)) ||
      (rc = d2h_slots(env, env->d.return_sum, r, st)) || (rc = d2h_slots(env, env->d.first_event, fe, st)) ||
      (rc = d2h_slots(env, env->d.first_ret, fr, st)) || (rc = d2h_slots(env, env->d.first_steps, fs, st)))
    return rc;
  SP_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < env->n; ++i) {
    const int64_t s = env->slot_of_env[i];
    if (episodes) episodes[i] = e[s];
    if (arrivals) arrivals[i] = a[s];
    if (return_sum) return_sum[i] = r[s];
    if (first_event) first_event[i] = fe[s];
    if (first_return) first_return[i] = fr[s];
    if (first_steps) first_steps[i] = fs[s];
  }
  return SP_OK;
}

int sp_env_recent_returns_keyed(SpEnv* env, double* out256, uint64_t* keys256, int32_t* n_out,
                                void* stream);

int sp_env_recent_returns(SpEnv* env, double* out256, int32_t* n_out, void* stream) {
  return sp_env_recent_returns_keyed(env, out256, nullptr, n_out, stream);
}

int sp_env_recent_returns_keyed(SpEnv* env, double* out256, uint64_t* keys256, int32_t* n_out,
                                void* stream) {
  if (!env || !out256 || !n_out) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long count = 0;
  SP_CUDA(cudaMemcpyAsync(&count, env->d.rec_count, 8, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  const uint64_t cap = env->d.rec_cap;
  const uint64_t valid = std::min<uint64_t>(count, cap);
  std::vector<double> ret(cap);
  std::vector<uint64_t> key(cap);
  SP_CUDA(cudaMemcpyAsync(ret.data(), env->d.rec_ret, 8 * cap, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaMemcpyAsync(key.data(), env->d.rec_key, 8 * cap, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  // entries written in the last `valid` reservations; order by (step, env)
  std::vector<std::pair<uint64_t, double>> items;
  items.reserve(valid);
  for (uint64_t k = count - valid; k < count; ++k) items.emplace_back(key[k % cap], ret[k % cap]);
  std::sort(items.begin(), items.end(),
            [](const std::pair<uint64_t, double>& x, const std::pair<uint64_t, double>& y) {
              return x.first < y.first;
            });
  const size_t take = std::min<size_t>(256, items.size());
  for (size_t i = 0; i < take; ++i) {
    const auto& it = items[items.size() - take + i];
    out256[i] = it.second;
    if (keys256)  // (step << 32) | global env id: merges across shards (dist.py)
      keys256[i] = (it.first & ~0xffffffffull) |
                   (uint64_t)(uint32_t)((it.first & 0xffffffffull) + (uint64_t)env->d.env_id_offset);
  }
  *n_out = (int32_t)take;
  return SP_OK;
}

int sp_env_stats_reset(SpEnv* env, int clear_recent, void* stream) {
  if (!env) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  SP_CUDA(cudaMemsetAsync(env->d.episodes, 0, 8 * env->n, st));
  SP_CUDA(cudaMemsetAsync(env->d.arrivals, 0, 8 * env->n, st));
  SP_CUDA(cudaMemsetAsync(env->d.return_sum, 0, 8 * env->n, st));
  if (clear_recent) SP_CUDA(cudaMemsetAsync(env->d.rec_count, 0, 8, st));
  return SP_OK;
}

int sp_env_first_pending(SpEnv* env, int64_t* host_count, void* stream) {
  if (!env || !host_count) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  cudaStream_t st = (cudaStream_t)stream;
  if (!env->d_count) {
    unsigned long long* p = nullptr;
    const int rc = env->alloc(&p, 1);
    if (rc != SP_OK) return rc;
    env->d_count = p;
  }
  SP_CUDA(cudaMemsetAsync(env->d_count, 0, 8, st));
  count_pending_kernel<<<grid_for(env->n, 256), 256, 0, st>>>(env->d.first_event, env->n,
                                                              env->d_count);
  SP_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  SP_CUDA(cudaMemcpyAsync(&h, env->d_count, 8, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  *host_count = (int64_t)h;
  return SP_OK;
}

int sp_env_stats_totals(SpEnv* env, double* dev_out3, void* stream) {
  if (!env || !dev_out3) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  stats_totals_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(env->d.episodes, env->d.arrivals,
                                                           env->d.return_sum, env->n, dev_out3);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_env_read_state(SpEnv* env, int field, double* host_out, void* stream) {
  if (!env || !host_out) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  const EnvDev& d = env->d;
  std::vector<double> tmp(env->n);
  const double* f64 = nullptr;
  switch (field) {
    case 0: f64 = d.x; break;
    case 1: f64 = d.y; break;
    case 2: f64 = d.h; break;
    case 3: f64 = d.vl; break;
    case 4: f64 = d.va; break;
    case 5: f64 = d.sx; break;
    case 6: f64 = d.sy; break;
    case 7: f64 = d.pk; break;
    case 8: f64 = d.pdt; break;
    case 10: f64 = d.pvl; break;
    case 11: f64 = d.pva; break;
    case 12: f64 = d.psig; break;
    case 16: f64 = d.ret; break;
    case 17: f64 = d.c0; break;
    case 18: f64 = d.s0; break;
    default: break;
  }
  if (f64) {
    SP_CUDA(cudaMemcpyAsync(tmp.data(), f64, 8 * env->n, cudaMemcpyDeviceToHost, st));
  } else if (field == 9 || field == 13) {
    std::vector<int32_t> v(env->n);
    SP_CUDA(cudaMemcpyAsync(v.data(), field == 9 ? d.delay : d.step, 4 * env->n, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < env->n; ++s) tmp[s] = v[s];
  } else if (field == 14) {
    std::vector<uint8_t> v(env->n);
    SP_CUDA(cudaMemcpyAsync(v.data(), d.needs_reset, env->n, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < env->n; ++s) tmp[s] = v[s];
  } else if (field == 15) {
    std::vector<uint64_t> v(env->n);
    SP_CUDA(cudaMemcpyAsync(v.data(), d.ctr, 8 * env->n, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < env->n; ++s) tmp[s] = (double)v[s];
  } else {
    return fail(SP_EINVAL, "unknown state field");
  }
  SP_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < env->n; ++i) host_out[i] = tmp[env->slot_of_env[i]];
  return SP_OK;
}

int sp_env_read_fifo(SpEnv* env, uint64_t* host_out, void* stream) {
  if (!env || !host_out) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = env->n;
  std::vector<uint64_t> h((size_t)(4 * n));
  SP_CUDA(cudaMemcpyAsync(h.data(), env->d.hist, 8 * 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = env->slot_of_env[i];
    for (int w = 0; w < 4; ++w) host_out[4 * i + w] = h[(size_t)(w * n + s)];
  }
  return SP_OK;
}

int sp_env_write_state(SpEnv* env, int field, const double* host_in, void* stream) {
  if (!env || !host_in) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  cudaStream_t st = (cudaStream_t)stream;
  const EnvDev& d = env->d;
  double* dst = nullptr;
  switch (field) {
    case 0: dst = d.x; break;
    case 1: dst = d.y; break;
    case 2: dst = d.h; break;
    case 3: dst = d.vl; break;
    case 4: dst = d.va; break;
    case 5: dst = d.sx; break;
    case 6: dst = d.sy; break;
    case 17: dst = d.c0; break;
    case 18: dst = d.s0; break;
    default: return fail(SP_EINVAL, "field is not writable");
  }
  std::vector<double> tmp(env->n);
  for (int64_t i = 0; i < env->n; ++i) tmp[env->slot_of_env[i]] = host_in[i];
  SP_CUDA(cudaMemcpyAsync(dst, tmp.data(), 8 * env->n, cudaMemcpyHostToDevice, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_env_reset_lanes(SpEnv* env, const uint8_t* mask, float* states, void* stream) {
  if (!env || !mask || !states) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  StepArgs a{};
  a.mode = MODE_RESET_LANES;
  a.reset_mask = mask;
  a.states = states;
  return launch_env(env, a, (cudaStream_t)stream);
}

int sp_env_map_info(SpEnv* env, int64_t* slot_of_env, int64_t* smem_bytes, int32_t* threads,
                    int32_t* ctas) {
  if (!env) return fail(SP_EINVAL, "null argument");
  if (slot_of_env) std::memcpy(slot_of_env, env->slot_of_env.data(), 8 * env->n);
  if (smem_bytes) *smem_bytes = (int64_t)env->smem;
  if (threads) *threads = env->threads;
  if (ctas) *ctas = env->grid;
  return SP_OK;
}

int sp_env_launch_info(SpEnv* env, int64_t* cuts, uint32_t* cta_cycles) {
  if (!env) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  SP_CUDA(cudaDeviceSynchronize());
  if (cuts) SP_CUDA(cudaMemcpy(cuts, env->d.cta_begin, 8 * (size_t)(env->grid + 1), cudaMemcpyDeviceToHost));
  if (cta_cycles) SP_CUDA(cudaMemcpy(cta_cycles, env->d.cta_cyc, 4 * (size_t)env->grid, cudaMemcpyDeviceToHost));
  return SP_OK;
}

int sp_env_scan(SpEnv* env, int64_t n, const int64_t* query_offsets, const double* x,
                const double* y, const double* heading, double* ranges, int32_t* hit_cell,
                void* stream) {
  if (!env || !query_offsets || !x || !y || !heading || !ranges) return fail(SP_EINVAL, "null argument");
  if (n < 1) return SP_OK;
  if (query_offsets[0] != 0 || query_offsets[env->n_maps] != n)
    return fail(SP_EINVAL, "query_offsets must span [0, n)");
  DevDeviceGuard guard(env->device);
  std::lock_guard<std::mutex> lk(env->mu);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int64_t> off(query_offsets, query_offsets + env->n_maps + 1);
  Plan plan = plan_launch(env, off, false);
  EnvDev d = env->d;
  apply_plan(plan, d);
  d.D = 0;  // chunk layout without staging rows
  const size_t nq = off.size(), nc = plan.cta_begin.size();
  // stage the offsets through pinned memory; wait only for the previous copy
  SP_CUDA(cudaEventSynchronize(env->scan_copied));
  std::memcpy(env->h_scan, off.data(), 8 * nq);
  std::memcpy(env->h_scan + nq, plan.cta_begin.data(), 8 * nc);
  SP_CUDA(cudaMemcpyAsync(env->d_scan, env->h_scan, 8 * (nq + nc), cudaMemcpyHostToDevice, st));
  SP_CUDA(cudaEventRecord(env->scan_copied, st));
  ScanArgs q{n, env->d_scan + nq, env->d_scan, x, y, heading, ranges, hit_cell};
  if (d.smem_maps)
    env_scan_kernel<true><<<plan.grid, plan.threads, plan.smem, st>>>(d, q);
  else
    env_scan_kernel<false><<<plan.grid, plan.threads, plan.smem, st>>>(d, q);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SP_ECUDA, std::string("env_scan_kernel: ") + cudaGetErrorString(e));
  return SP_OK;
}

// ------------------------------------------------------------- op seam ----

int sp_cast_rays(const uint8_t* occ, const double* edt, int64_t n_maps, int64_t height,
                 int64_t width, const int64_t* map_idx, const double* px, const double* py,
                 const double* dirx, const double* diry, int64_t n, double cell, double max_range,
                 double* out, void* stream) {
  if (n < 1) return SP_OK;
  if (!occ || !edt || !map_idx || !px || !py || !dirx || !diry || !out || n_maps < 1)
    return fail(SP_EINVAL, "null argument");
  cast_rays_exact_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      occ, edt, height, width, map_idx, px, py, dirx, diry, n, cell, max_range, out);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_disc_collides(const uint8_t* occ, int64_t n_maps, int64_t height, int64_t width,
                     const int64_t* map_idx, const double* px, const double* py,
                     const double* radius, int64_t n, double cell, uint8_t* out, void* stream) {
  if (n < 1) return SP_OK;
  if (!occ || !map_idx || !px || !py || !radius || !out || n_maps < 1)
    return fail(SP_EINVAL, "null argument");
  disc_collides_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      occ, height, width, map_idx, px, py, radius, n, cell, out);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// -------------------------------------------------------------- replay -----
int sp_rb_create(int64_t capacity, int32_t state_dim, int device, SpReplay** out) {
  if (capacity < 1) return fail(SP_EINVAL, "capacity must be positive");  // replay.py:33-34
  if (state_dim < 1 || !out) return fail(SP_EINVAL, "bad state_dim");
  DevDeviceGuard guard(device);
  SpReplay* rb = new SpReplay();
  rb->device = device;
  rb->cap = capacity;
  rb->dim = state_dim;
  const size_t rows = (size_t)capacity;
  if (cudaMalloc(&rb->s, rows * state_dim * 4) != cudaSuccess ||
      cudaMalloc(&rb->s2, rows * state_dim * 4) != cudaSuccess ||
      cudaMalloc(&rb->r, rows * 4) != cudaSuccess || cudaMalloc(&rb->a, rows * 8) != cudaSuccess ||
      cudaMalloc(&rb->dn, rows) != cudaSuccess || cudaMalloc(&rb->d_size, 8) != cudaSuccess ||
      cudaMemset(rb->d_size, 0, 8) != cudaSuccess) {
    delete rb;
    return fail(SP_ENOMEM, "replay allocation failed");
  }
  cudaMemset(rb->s, 0, rows * state_dim * 4);
  cudaMemset(rb->s2, 0, rows * state_dim * 4);
  cudaMemset(rb->r, 0, rows * 4);
  cudaMemset(rb->a, 0, rows * 8);
  cudaMemset(rb->dn, 0, rows);
  cudaDeviceSynchronize();
  *out = rb;
  return SP_OK;
}

int sp_rb_destroy(SpReplay* rb) {
  if (!rb) return SP_OK;
  DevDeviceGuard guard(rb->device);
  cudaDeviceSynchronize();
  delete rb;
  return SP_OK;
}

int sp_rb_append(SpReplay* rb, const float* states, const int64_t* actions, const void* rewards,
                 int reward_is_f64, const float* next_states, const uint8_t* dones, int64_t n,
                 void* stream) {
  if (!rb) return fail(SP_EINVAL, "null argument");
  if (n > rb->cap)
    return fail(SP_EINVAL, "batch of " + std::to_string(n) + " exceeds capacity " + std::to_string(rb->cap));
  if (n < 1) return SP_OK;
  if (!states || !actions || !rewards || !next_states || !dones) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(rb->device);
  std::lock_guard<std::mutex> lk(rb->mu);
  const int64_t new_size = std::min(rb->size + n, rb->cap);
  const int64_t D = rb->dim, n1 = std::min(n, rb->cap - rb->cursor);
  AppendSeg g{};
  auto add = [&](float* dst, const float* src, int64_t count) {
    if (count <= 0) return;
    const int k = g.nseg++;
    const int64_t head = std::min<int64_t>(count, ((16 - ((uintptr_t)dst & 15)) & 15) / 4);
    g.dst[k] = dst;
    g.src[k] = src;
    g.head[k] = head;
    g.nvec[k] = (count - head) / 4;
    g.count[k] = count;
    g.vend[k] = (k ? g.vend[k - 1] : 0) + g.nvec[k];
  };
  add(rb->s + rb->cursor * D, states, n1 * D);
  add(rb->s2 + rb->cursor * D, next_states, n1 * D);
  add(rb->s, states + n1 * D, (n - n1) * D);
  add(rb->s2, next_states + n1 * D, (n - n1) * D);
  // kAppendU vectors (and rows) per thread in one pass, <= 8 CTAs per SM
  const int64_t items = std::max<int64_t>(g.vend[g.nseg - 1], n);
  const int64_t thr = std::max<int64_t>(1, (items + kAppendU - 1) / kAppendU);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((thr + 255) / 256, 148 * 8));
  rb_append_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      g, rb->a, rb->r, rb->dn, rb->cap, rb->cursor, actions, rewards, reward_is_f64, dones, n,
      rb->d_size, new_size);
  SP_CUDA(cudaGetLastError());
  rb->cursor = (rb->cursor + n) % rb->cap;  // replay.py:66-67
  rb->size = new_size;
  return SP_OK;
}

int sp_rb_sample(SpReplay* rb, int64_t batch, uint64_t seed, uint32_t stream_id, uint64_t ctr,
                 float* states, int64_t* actions, float* rewards, float* next_states,
                 uint8_t* dones, int64_t* idx_out, void* stream) {
  if (!rb) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(rb->device);
  std::lock_guard<std::mutex> lk(rb->mu);
  if (rb->size < batch)  // replay.py:73-75
    return fail(SP_ENOTREADY, "buffer holds " + std::to_string(rb->size) + " transitions, need " +
                                  std::to_string(batch));
  if (batch < 1) return SP_OK;
  if (!states || !actions || !rewards || !next_states || !dones) return fail(SP_EINVAL, "null argument");
  const int blocks = (int)((batch + 7) / 8);  // one warp per row
  rb_sample_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      rb->s, rb->a, rb->r, rb->s2, rb->dn, rb->dim, rb->size, batch, seed, stream_id, ctr, states,
      actions, rewards, next_states, dones, idx_out, nullptr, nullptr);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_rb_sample_dev(SpReplay* rb, int64_t batch, uint64_t seed, uint32_t stream_id,
                     uint64_t* d_ctr, float* states, int64_t* actions, float* rewards,
                     float* next_states, uint8_t* dones, int64_t* idx_out, void* stream) {
  if (!rb || !d_ctr) return fail(SP_EINVAL, "null argument");
  if (batch < 1) return SP_OK;
  if (!states || !actions || !rewards || !next_states || !dones) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(rb->device);
  const int blocks = (int)((batch + 7) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  rb_sample_kernel<<<blocks, 256, 0, st>>>(rb->s, rb->a, rb->r, rb->s2, rb->dn, rb->dim, 0, batch,
                                           seed, stream_id, 0, states, actions, rewards,
                                           next_states, dones, idx_out, rb->d_size, d_ctr);
  SP_CUDA(cudaGetLastError());
  rb_ctr_advance_kernel<<<1, 1, 0, st>>>(d_ctr, batch);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_rb_size(SpReplay* rb, int64_t* size, int64_t* cursor) {
  if (!rb) return fail(SP_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(rb->mu);
  if (size) *size = rb->size;
  if (cursor) *cursor = rb->cursor;
  return SP_OK;
}

int sp_rb_gather(SpReplay* rb, float* states, int64_t* actions, float* rewards, float* next_states,
                 uint8_t* dones, void* stream) {
  if (!rb) return fail(SP_EINVAL, "null argument");
  DevDeviceGuard guard(rb->device);
  std::lock_guard<std::mutex> lk(rb->mu);
  if (rb->size < 1) return SP_OK;
  const int64_t flat = rb->size * rb->dim;
  rb_gather_kernel<<<grid_for(flat, 256), 256, 0, (cudaStream_t)stream>>>(
      rb->s, rb->a, rb->r, rb->s2, rb->dn, rb->dim, rb->size, states, actions, rewards,
      next_states, dones);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_philox_fill(int64_t n, uint64_t seed, uint32_t lane, uint32_t tag, uint64_t ctr0,
                   int kind, double lo, double hi, void* out, void* stream) {
  if (n < 1) return SP_OK;
  if (!out || (kind != 0 && kind != 1)) return fail(SP_EINVAL, "bad arguments");
  if (kind == 1 && !(hi > lo)) return fail(SP_EINVAL, "integers: high <= low");
  philox_fill_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, seed, lane, tag, ctr0,
                                                                        kind, lo, hi, out);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_random_actions(int64_t n, uint64_t seed, int64_t env_id0, int64_t step, int32_t n_actions,
                      int64_t* actions, void* stream) {
  if (n < 1) return SP_OK;
  if (!actions || n_actions < 1) return fail(SP_EINVAL, "bad arguments");
  random_actions_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, seed, env_id0, step,
                                                                           n_actions, actions);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_adam_step(int n_tensors, float* const* params, const float* const* grads, float* const* m,
                 float* const* v, const int64_t* numels, double* step_dev, int64_t step_host,
                 const float* gate, double lr, double beta1, double beta2, double eps,
                 void* stream) {
  if (n_tensors < 1 || n_tensors > SP_ADAM_MAX || !params || !grads || !m || !v || !numels)
    return fail(SP_EINVAL, "adam: bad tensor list");
  if (!step_dev && step_host < 1) return fail(SP_EINVAL, "adam: step must be >= 1");
  AdamTensors T;
  int64_t acc = 0;
  for (int k = 0; k < n_tensors; ++k) {
    if (numels[k] < 1 || !params[k] || !grads[k] || !m[k] || !v[k])
      return fail(SP_EINVAL, "adam: empty or null tensor");
    T.p[k] = params[k];
    T.g[k] = grads[k];
    T.m[k] = m[k];
    T.v[k] = v[k];
    acc += numels[k];
    T.end[k] = acc;
  }
  T.n = n_tensors;
  cudaStream_t s = (cudaStream_t)stream;
  adam_kernel<<<grid_for(acc, 256), 256, 0, s>>>(T, step_dev, step_host, gate, lr, beta1, beta2,
                                                  eps);
  SP_CUDA(cudaGetLastError());
  if (step_dev) {
    adam_tick_kernel<<<1, 1, 0, s>>>(step_dev, gate);
    SP_CUDA(cudaGetLastError());
  }
  return SP_OK;
}

// rows per CTA of ddqn_rows_kernel: 2 (128 CTAs at B = 256) measured best
// (per-CTA serial work halves; the extra weight staging streams from L2)
static int learn_tr(int64_t batch) { return batch % 2 == 0 ? 2 : 1; }

static size_t ddqn_rows_smem(const int32_t* sz, int64_t batch) {
  return learn_tr(batch) == 2 ? learn_smem_bytes<2>(sz[0], sz[1], sz[2], sz[3])
                              : learn_smem_bytes<1>(sz[0], sz[1], sz[2], sz[3]);
}

int64_t sp_ddqn_scratch_floats(const int32_t* sz, int64_t batch) {
  if (!sz || batch < 1) return -1;
  // the fused kernels' limits (shared memory for the staged layers, tiles)
  if (sz[0] < 1 || sz[0] > kLearnMaxD0 || sz[1] < 1 || sz[1] > kLearnMaxH || sz[2] < 1 ||
      sz[2] > kLearnMaxH || sz[3] < 1 || sz[3] > kLearnMaxA || ddqn_rows_smem(sz, batch) > 227 * 1024 ||
      (size_t)batch * (kGradTK + kGradTJ) * 4 > 200 * 1024)
    return -1;
  const int64_t tiles = batch / learn_tr(batch);
  // a1, d1 (B x H1), a2, d2 (B x H2), dq (B x A), loss partials (tiles x 2)
  return batch * (2 * (int64_t)sz[1] + 2 * (int64_t)sz[2] + sz[3]) + 2 * tiles;
}

int sp_ddqn_update(const SpMlp* on, const SpMlp* tg, const float* s, const int64_t* a,
                   const float* r, const float* s2, const uint8_t* d, int64_t batch, float gamma,
                   float* const* m, float* const* v, double* step_dev, double lr, double beta1,
                   double beta2, double eps, float* scratch, int64_t scratch_floats,
                   float* stats_out, void* stream) {
  if (!on || !tg || !s || !a || !r || !s2 || !d || !m || !v || !step_dev || !scratch || !stats_out)
    return fail(SP_EINVAL, "ddqn_update: null argument");
  const int D0 = on->sizes[0], H1 = on->sizes[1], H2 = on->sizes[2], A = on->sizes[3];
  for (int k = 0; k < 4; ++k)
    if (tg->sizes[k] != on->sizes[k]) return fail(SP_EINVAL, "ddqn_update: online/target shapes differ");
  if (D0 < 1 || D0 > kLearnMaxD0 || H1 < 1 || H1 > kLearnMaxH || H2 < 1 || H2 > kLearnMaxH ||
      A < 1 || A > kLearnMaxA)
    return fail(SP_EINVAL, "ddqn_update: unsupported layer sizes");
  for (int l = 0; l < 3; ++l)
    if (((uintptr_t)on->W[l] | (uintptr_t)tg->W[l]) & 15)
      return fail(SP_EINVAL, "ddqn_update: weights must be 16-byte aligned");
  if (((int64_t)D0 * H1) % 4 || ((int64_t)H1 * H2) % 4 || ((int64_t)H2 * A) % 4)
    return fail(SP_EINVAL, "ddqn_update: each weight matrix must hold a multiple of 4 floats");
  if (batch < 1 || batch > (1 << 24)) return fail(SP_EINVAL, "ddqn_update: bad batch size");
  const int64_t need = sp_ddqn_scratch_floats(on->sizes, batch);
  if (need < 0) return fail(SP_EINVAL, "ddqn_update: layer sizes / batch exceed the fused kernels");
  if (scratch_floats < need) return fail(SP_EINVAL, "ddqn_update: scratch too small");
  const int TR = learn_tr(batch);
  const int tiles = (int)(batch / TR);
  LearnArgs la{};
  for (int l = 0; l < 3; ++l) {
    la.on.W[l] = on->W[l];
    la.on.b[l] = on->b[l];
    la.tgt.W[l] = tg->W[l];
    la.tgt.b[l] = tg->b[l];
  }
  la.s = s; la.a = a; la.r = r; la.s2 = s2; la.d = d;
  la.B = (int)batch; la.D0 = D0; la.H1 = H1; la.H2 = H2; la.A = A;
  la.a1 = scratch;
  la.d1 = la.a1 + batch * H1;
  la.a2 = la.d1 + batch * H1;
  la.d2 = la.a2 + batch * H2;
  la.dq = la.d2 + batch * H2;
  la.lpart = la.dq + batch * A;
  la.gamma = gamma;
  cudaStream_t st = (cudaStream_t)stream;
  if (TR == 2) {
    const size_t sm = learn_smem_bytes<2>(D0, H1, H2, A);
    SP_CUDA(cudaFuncSetAttribute(ddqn_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
    ddqn_rows_kernel<2><<<tiles, kLearnThreads, sm, st>>>(la);
  } else {
    const size_t sm = learn_smem_bytes<1>(D0, H1, H2, A);
    SP_CUDA(cudaFuncSetAttribute(ddqn_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
    ddqn_rows_kernel<1><<<tiles, kLearnThreads, sm, st>>>(la);
  }
  SP_CUDA(cudaGetLastError());
  AdamTensors T;
  const float* ps[6] = {on->W[0], on->W[1], on->W[2], on->b[0], on->b[1], on->b[2]};
  const int64_t n[6] = {(int64_t)D0 * H1, (int64_t)H1 * H2, (int64_t)H2 * A, H1, H2, A};
  int64_t acc = 0;
  for (int k = 0; k < 6; ++k) {
    if (!m[k] || !v[k]) return fail(SP_EINVAL, "ddqn_update: null moment tensor");
    T.p[k] = const_cast<float*>(ps[k]);
    T.g[k] = nullptr;
    T.m[k] = m[k];
    T.v[k] = v[k];
    acc += n[k];
    T.end[k] = acc;
  }
  T.n = 6;
  GradTiles gt{};
  const int dims[3][2] = {{D0, H1}, {H1, H2}, {H2, A}};
  for (int tk = 0; tk < 3; ++tk)
    for (int k0 = 0; k0 < dims[tk][0]; k0 += kGradTK)
      for (int j0 = 0; j0 < dims[tk][1]; j0 += kGradTJ) {
        if (gt.n >= kMaxGradTiles) return fail(SP_EINVAL, "ddqn_update: too many gradient tiles");
        gt.tensor[gt.n] = (uint8_t)tk;
        gt.k0[gt.n] = (int16_t)k0;
        gt.j0[gt.n] = (int16_t)j0;
        ++gt.n;
      }
  const size_t gsm = sizeof(float) * (size_t)batch * (kGradTK + kGradTJ);
  if (gsm > 200 * 1024) return fail(SP_EINVAL, "ddqn_update: batch too large for the gradient tiles");
  SP_CUDA(cudaFuncSetAttribute(ddqn_grad_adam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gsm));
  ddqn_grad_adam_kernel<<<gt.n, 256, gsm, st>>>(la, T, gt, tiles, step_dev, lr, beta1, beta2, eps,
                                                stats_out);
  SP_CUDA(cudaGetLastError());
  adam_tick_stats_kernel<<<1, 1, 0, st>>>(step_dev, stats_out);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_actor_select(const SpMlp* net, const float* states, int64_t n, int64_t env0,
                    const SpVem* vem, int64_t t_step, uint64_t seed, uint32_t lane, uint32_t tag,
                    uint64_t ctr, int64_t* actions, float* q_out, void* stream) {
  if (!net || !vem || (n > 0 && (!states || !actions))) return fail(SP_EINVAL, "null argument");
  if (n < 1) return SP_OK;
  const int D0 = net->sizes[0], H1 = net->sizes[1], H2 = net->sizes[2], A = net->sizes[3];
  if (D0 < 1 || D0 > kActMaxD0 || H1 < 1 || H1 > kActMaxH || H2 < 1 || H2 > kActMaxH || A < 1 ||
      A > kActMaxA)
    return fail(SP_EINVAL, "actor: unsupported layer sizes");
  if ((D0 * H1) % 4 || (H1 * H2) % 4 || (H2 * A) % 4)
    return fail(SP_EINVAL, "actor: each weight matrix must hold a multiple of 4 floats");
  for (int l = 0; l < 3; ++l)
    if (!net->W[l] || !net->b[l] || ((uintptr_t)net->W[l] & 15))
      return fail(SP_EINVAL, "actor: weights must be 16-byte aligned device tensors");
  if (!(vem->n_envs >= 1 && 1 <= vem->or_final && vem->or_final <= vem->or_init &&
        vem->or_init <= vem->n_envs && vem->decay_steps >= 1 && 0.0 <= vem->e_min &&
        vem->e_min <= vem->e_max && vem->e_max <= 1.0))
    return fail(SP_EINVAL, "actor: bad VEM schedule");  // vem.py:28-35
  if (env0 < 0 || env0 + n > vem->n_envs) return fail(SP_EINVAL, "actor: rows outside the VEM copies");
  int dev = 0;
  SP_CUDA(cudaGetDevice(&dev));
  int optin = 0, n_sm = 0;
  SP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  SP_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  int rows = 32;
  while (rows > 4 && actor_smem_bytes(D0, H1, H2, A, rows) > (size_t)optin) rows /= 2;
  const size_t sm = actor_smem_bytes(D0, H1, H2, A, rows);
  if (sm > (size_t)optin) return fail(SP_EINVAL, "actor: weights do not fit in shared memory");
  ActorArgs a{};
  for (int l = 0; l < 3; ++l) {
    a.W[l] = net->W[l];
    a.b[l] = net->b[l];
  }
  a.D0 = D0; a.H1 = H1; a.H2 = H2; a.A = A; a.L0 = pad4(D0); a.rows = rows;
  a.states = states; a.n = n; a.env0 = env0;
  a.vem = VemDev{vem->n_envs, vem->or_init, vem->or_final, vem->decay_steps, vem->e_min,
                 vem->e_max};
  a.t_step = t_step; a.seed = seed; a.lane = lane; a.tag = tag; a.ctr = ctr;
  a.actions = actions; a.q_out = q_out;
  SP_CUDA(cudaFuncSetAttribute(actor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int64_t tiles = (n + rows - 1) / rows;
  const int grid = (int)std::min<int64_t>(tiles, n_sm);
  actor_kernel<<<grid, kActThreads, sm, (cudaStream_t)stream>>>(a);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

#ifdef SP_TIMING
// debug builds only (not part of include/sparrow.h): per-CTA phase stamps
int sp_debug_read_lane(unsigned long long* out, int n_ctas) {
  (void)n_ctas;
  SP_CUDA(cudaMemcpyFromSymbol(out, g_sp_lane, sizeof(unsigned long long) * 5 * 148 * 768));
  return SP_OK;
}
int sp_debug_read_ts(unsigned long long* out, int n_ctas) {
  SP_CUDA(cudaDeviceSynchronize());
  SP_CUDA(cudaMemcpyFromSymbol(out, g_sp_ts, sizeof(unsigned long long) * kTs * (size_t)n_ctas));
  return SP_OK;
}
#endif

}  // extern "C"
