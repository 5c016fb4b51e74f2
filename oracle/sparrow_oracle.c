/*
 * sparrow_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A scalar C restatement of the reference's Sparrow hot path
 * (color-rl 0.1.0 under /root/reference/pkg/src/color_rl), used ONLY as the
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * The product (paper_2305_04180_b200/) never links, loads or calls this file.
 *
 * Every function names the reference lines it restates.  Floating point is
 * IEEE double with the reference's operation order; compile with
 * -ffp-contract=off so no FMA contraction changes rounding.  Randomness is the
 * counter-based Philox4x32-10 stream contract of DESIGN.md section "RNG
 * contract" (the reference's numpy PCG64 streams are replaced by that
 * contract on both sides of every parity test; see oracle/philox_shim.py,
 * which drives the UNMODIFIED reference with the same streams).
 *
 * Parity pin: tests/test_oracle_vs_reference.py runs the real reference
 * (oracle/_ref, built by oracle/build_ref.sh) and this file on identical
 * seeds/inputs; they agree bit for bit except quantities that go through
 * atan2 / log (numpy's SIMD atan2/log differ from glibc in the last ulp),
 * which agree to <1e-12 relative.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_EACTION 2
#define OR_EEPISODE 3
#define OR_EMAP 4

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 + draw mappings                  */
/* ------------------------------------------------------------------------ */

void or_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

typedef struct {
  uint64_t seed;
  uint32_t lane; /* global env id (or stream id) */
  uint32_t tag;  /* stream family */
  uint64_t ctr;  /* next block */
} OrStream;

static void or_block(OrStream* s, uint32_t out[4]) {
  uint32_t c[4] = {(uint32_t)s->ctr, (uint32_t)(s->ctr >> 32), s->lane, s->tag};
  or_philox4x32_10(c, (uint32_t)s->seed, (uint32_t)(s->seed >> 32), out);
  s->ctr += 1;
}

static uint64_t or_word64(const uint32_t b[4]) { return ((uint64_t)b[1] << 32) | b[0]; }

/* numpy Generator.uniform(lo, hi): lo + (hi - lo) * u53 */
static double or_uniform(OrStream* s, double lo, double hi) {
  uint32_t b[4];
  or_block(s, b);
  double u = (double)(or_word64(b) >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * u;
}

/* numpy Generator.integers(lo, hi) (hi exclusive): lo + mulhi64(w, hi - lo) */
static int64_t or_integers(OrStream* s, int64_t lo, int64_t hi) {
  uint32_t b[4];
  or_block(s, b);
  unsigned __int128 p = (unsigned __int128)or_word64(b) * (uint64_t)(hi - lo);
  return lo + (int64_t)(uint64_t)(p >> 64);
}

/* Standard normals, 4 per block: Box-Muller on (x0, x1) and (x2, x3). */
static void or_normals(OrStream* s, double* z, int n) {
  for (int j = 0; j < n; j += 4) {
    uint32_t b[4];
    or_block(s, b);
    for (int h = 0; h < 2; ++h) {
      double u1 = ((double)b[2 * h] + 1.0) * 0x1.0p-32;
      double u2 = (double)b[2 * h + 1] * 0x1.0p-32;
      double r = sqrt(-2.0 * log(u1));
      double a = 2.0 * M_PI * u2;
      if (j + 2 * h < n) z[j + 2 * h] = r * cos(a);
      if (j + 2 * h + 1 < n) z[j + 2 * h + 1] = r * sin(a);
    }
  }
}

/* exported for the numpy shim's self-check */
void or_stream_draw(uint64_t seed, uint32_t lane, uint32_t tag, uint64_t ctr, int kind,
                    double lo, double hi, int n, double* out) {
  OrStream s = {seed, lane, tag, ctr};
  if (kind == 0) {
    for (int i = 0; i < n; ++i) out[i] = or_uniform(&s, lo, hi);
  } else if (kind == 1) {
    for (int i = 0; i < n; ++i) out[i] = (double)or_integers(&s, (int64_t)lo, (int64_t)hi);
  } else {
    or_normals(&s, out, n);
  }
}

/* ------------------------------------------------------------------------ */
/* Kernels: restates kernels/_cy.pyx (bit-identical twin of kernels/_py.py)  */
/* ------------------------------------------------------------------------ */

#define JUMP_MIN_CELLS 2.5 /* _cy.pyx:15 */
#define JUMP_MARGIN 1.5    /* _cy.pyx:16 */

/* cast_rays, _cy.pyx:19-106.  Optional hit_cell[r] = iy*W+ix of the cell the
 * march stopped in (-1 when it stopped on max_range or outside the grid). */
static double or_cast_one(const uint8_t* occ, const double* edt, int64_t H, int64_t W, double x0,
                          double y0, double dx, double dy, double cell, double max_range,
                          int64_t* hit_cell, int64_t* n_iter) {
  const double INF = INFINITY;
  int64_t ix = (int64_t)floor(x0 / cell);
  int64_t iy = (int64_t)floor(y0 / cell);
  int64_t it = 0;
  if (hit_cell) *hit_cell = -1;
  if (n_iter) *n_iter = 0;
  if (ix < 0 || ix >= W || iy < 0 || iy >= H) return 0.0; /* :37-39 */
  if (occ[iy * W + ix]) {                                  /* :40-42 */
    if (hit_cell) *hit_cell = iy * W + ix;
    return 0.0;
  }
  int64_t stepx = dx > 0 ? 1 : (dx < 0 ? -1 : 0); /* :43-44 */
  int64_t stepy = dy > 0 ? 1 : (dy < 0 ? -1 : 0);
  double tdx = dx != 0 ? cell / fabs(dx) : INF; /* :45-46 */
  double tdy = dy != 0 ? cell / fabs(dy) : INF;
  double tmx, tmy;
  if (dx > 0) tmx = ((double)(ix + 1) * cell - x0) / dx; /* :47-58 */
  else if (dx < 0) tmx = ((double)ix * cell - x0) / dx;
  else tmx = INF;
  if (dy > 0) tmy = ((double)(iy + 1) * cell - y0) / dy;
  else if (dy < 0) tmy = ((double)iy * cell - y0) / dy;
  else tmy = INF;
  double t = 0.0;
  double out = max_range;
  for (;;) { /* :61-105 */
    ++it;
    double clearance = edt[iy * W + ix];
    if (clearance > JUMP_MIN_CELLS) { /* EDT jump, :63-88 */
      double tj = t + (clearance - JUMP_MARGIN) * cell;
      double qx = x0 + tj * dx;
      double qy = y0 + tj * dy;
      ix = (int64_t)floor(qx / cell);
      iy = (int64_t)floor(qy / cell);
      if (dx > 0) tmx = ((double)(ix + 1) * cell - qx) / dx + tj;
      else if (dx < 0) tmx = ((double)ix * cell - qx) / dx + tj;
      else tmx = INF;
      if (dy > 0) tmy = ((double)(iy + 1) * cell - qy) / dy + tj;
      else if (dy < 0) tmy = ((double)iy * cell - qy) / dy + tj;
      else tmy = INF;
      t = tj;
      if (t > max_range) { out = max_range; break; }
      if (ix < 0 || ix >= W || iy < 0 || iy >= H) { out = t < max_range ? t : max_range; break; }
      continue;
    }
    if (tmx <= tmy) { /* DDA step with the x-first tie rule, :89-96 */
      t = tmx;
      tmx = tmx + tdx;
      ix = ix + stepx;
    } else {
      t = tmy;
      tmy = tmy + tdy;
      iy = iy + stepy;
    }
    if (t > max_range) { out = max_range; break; }
    if (ix < 0 || ix >= W || iy < 0 || iy >= H) { out = t < max_range ? t : max_range; break; }
    if (occ[iy * W + ix]) {
      out = t < max_range ? t : max_range;
      if (hit_cell && t <= max_range) *hit_cell = iy * W + ix;
      break;
    }
  }
  if (n_iter) *n_iter = it;
  return out;
}

void or_cast_rays(const uint8_t* occ, const double* edt, int64_t H, int64_t W,
                  const int64_t* map_idx, const double* px, const double* py, const double* dirx,
                  const double* diry, int64_t n, double cell, double max_range, double* out,
                  int64_t* hit_cell) {
  for (int64_t r = 0; r < n; ++r) {
    int64_t m = map_idx[r];
    out[r] = or_cast_one(occ + m * H * W, edt + m * H * W, H, W, px[r], py[r], dirx[r], diry[r],
                         cell, max_range, hit_cell ? hit_cell + r : NULL, NULL);
  }
}

/* Pure cell-by-cell DDA (no EDT jump): the traversal the ray-cells metric
 * counts; returns cells entered per ray. */
void or_count_dda_cells(const uint8_t* occ, int64_t H, int64_t W, const int64_t* map_idx,
                        const double* px, const double* py, const double* dirx, const double* diry,
                        int64_t n, double cell, double max_range, int64_t* cells) {
  for (int64_t r = 0; r < n; ++r) {
    const uint8_t* o = occ + map_idx[r] * H * W;
    double x0 = px[r], y0 = py[r], dx = dirx[r], dy = diry[r];
    int64_t ix = (int64_t)floor(x0 / cell), iy = (int64_t)floor(y0 / cell), c = 1;
    if (ix < 0 || ix >= W || iy < 0 || iy >= H || o[iy * W + ix]) { cells[r] = c; continue; }
    int64_t sx = dx > 0 ? 1 : (dx < 0 ? -1 : 0), sy = dy > 0 ? 1 : (dy < 0 ? -1 : 0);
    double tdx = dx != 0 ? cell / fabs(dx) : INFINITY, tdy = dy != 0 ? cell / fabs(dy) : INFINITY;
    double tmx = dx > 0 ? ((double)(ix + 1) * cell - x0) / dx
                        : (dx < 0 ? ((double)ix * cell - x0) / dx : INFINITY);
    double tmy = dy > 0 ? ((double)(iy + 1) * cell - y0) / dy
                        : (dy < 0 ? ((double)iy * cell - y0) / dy : INFINITY);
    for (;;) {
      double t;
      if (tmx <= tmy) { t = tmx; tmx += tdx; ix += sx; }
      else { t = tmy; tmy += tdy; iy += sy; }
      if (t > max_range) break;
      ++c;
      if (ix < 0 || ix >= W || iy < 0 || iy >= H || o[iy * W + ix]) break;
    }
    cells[r] = c;
  }
}

/* disc_collides, _cy.pyx:109-158 */
static int or_disc_one(const uint8_t* occ, int64_t H, int64_t W, double x, double y, double r,
                       double cell) {
  if (x - r < 0.0 || y - r < 0.0 || x + r > (double)W * cell || y + r > (double)H * cell)
    return 1; /* :124-126 */
  int64_t ix0 = (int64_t)floor((x - r) / cell); if (ix0 < 0) ix0 = 0; /* :128-135 */
  int64_t ix1 = (int64_t)floor((x + r) / cell); if (ix1 > W - 1) ix1 = W - 1;
  int64_t iy0 = (int64_t)floor((y - r) / cell); if (iy0 < 0) iy0 = 0;
  int64_t iy1 = (int64_t)floor((y + r) / cell); if (iy1 > H - 1) iy1 = H - 1;
  for (int64_t iy = iy0; iy <= iy1; ++iy) { /* :137-153 nearest-point test */
    for (int64_t ix = ix0; ix <= ix1; ++ix) {
      if (!occ[iy * W + ix]) continue;
      double lo = (double)ix * cell, hi = lo + cell;
      double nx = x > lo ? x : lo;
      if (nx > hi) nx = hi;
      lo = (double)iy * cell;
      hi = lo + cell;
      double ny = y > lo ? y : lo;
      if (ny > hi) ny = hi;
      double ddx = x - nx, ddy = y - ny;
      if (ddx * ddx + ddy * ddy <= r * r) return 1;
    }
  }
  return 0;
}

void or_disc_collides(const uint8_t* occ, int64_t H, int64_t W, const int64_t* map_idx,
                      const double* px, const double* py, const double* radius, int64_t n,
                      double cell, uint8_t* out) {
  for (int64_t k = 0; k < n; ++k)
    out[k] = (uint8_t)or_disc_one(occ + map_idx[k] * H * W, H, W, px[k], py[k], radius[k], cell);
}

/* ------------------------------------------------------------------------ */
/* Env: restates sim/core.py SimBatch + vecenv.py VecEnv                     */
/* ------------------------------------------------------------------------ */

#define OR_MAX_DELAY 64 /* params.py:20 */

typedef struct {
  /* config (params.py:124-151) */
  int32_t n_beams;
  double max_range, robot_radius, proximity;
  int32_t timeout_steps, spawn_attempts, auto_reset, n_actions;
  double action_table[32][2];
  /* maps (stacked like core.py:68-71) */
  int64_t n_maps, H, W;
  double cell;
  const uint8_t* occ;
  const double* edt;
  const double *goal_x, *goal_y, *goal_r, *plan_dist, *spawn; /* per map; spawn 4 per map */
  /* lanes */
  int64_t n;
  const int64_t* map_index;
  const double* ranges; /* per lane 12 doubles: k0 k1 dt0 dt1 d0 d1 vl0 vl1 va0 va1 s0 s1 */
  const double* offsets; /* n_beams, LidarConfig.beam_offsets() (params.py:132-133) */
  uint64_t seed;
  int64_t env_id_offset;
  /* SoA state (core.py:88-108) */
  double *x, *y, *heading, *vl, *va, *start_x, *start_y, *start_cos, *start_sin;
  double *pk, *pdt, *pvl, *pva, *psig;
  int64_t *pdelay, *step_count;
  uint8_t* needs_reset;
  double* last_scan; /* n * n_beams */
  double* qv;        /* pending queue ring: n * 65 * 2 */
  int32_t *qhead, *qlen;
  OrStream* rng;
  /* VecEnv bookkeeping (vecenv.py:76-80) */
  double* ep_return;
  int64_t *episodes, *arrivals;
  double* return_sum;
  int8_t* first_event;
  double* first_return;
  int64_t* first_steps;
  double recent[256];
  int64_t recent_count; /* total appended */
  /* scratch */
  double *scan_raw, *scan_min;
  /* hit cells (or_cast_one's hit_cell) of the scan behind the current states
   * row (cells_last) and of the last step's post-step scan (cells_store) */
  int64_t *cells_last, *cells_store;
  int err_lane;
} OrEnv;

static void* or_zalloc(size_t bytes) { return calloc(1, bytes ? bytes : 1); }

OrEnv* or_env_create(int32_t n_beams, double max_range, double robot_radius, double proximity,
                     int32_t timeout_steps, int32_t spawn_attempts, int32_t auto_reset,
                     int32_t n_actions, const double* action_table, int64_t n_maps, int64_t H,
                     int64_t W, double cell, const uint8_t* occ, const double* edt,
                     const double* goal_x, const double* goal_y, const double* goal_r,
                     const double* plan_dist, const double* spawn, int64_t n,
                     const int64_t* map_index, const double* ranges, const double* offsets,
                     int64_t env_id_offset) {
  OrEnv* e = (OrEnv*)or_zalloc(sizeof(OrEnv));
  e->n_beams = n_beams; e->max_range = max_range; e->robot_radius = robot_radius;
  e->proximity = proximity; e->timeout_steps = timeout_steps; e->spawn_attempts = spawn_attempts;
  e->auto_reset = auto_reset; e->n_actions = n_actions;
  for (int a = 0; a < n_actions && a < 32; ++a) {
    e->action_table[a][0] = action_table[2 * a];
    e->action_table[a][1] = action_table[2 * a + 1];
  }
  e->n_maps = n_maps; e->H = H; e->W = W; e->cell = cell; e->occ = occ; e->edt = edt;
  e->goal_x = goal_x; e->goal_y = goal_y; e->goal_r = goal_r; e->plan_dist = plan_dist;
  e->spawn = spawn; e->n = n; e->map_index = map_index; e->ranges = ranges; e->offsets = offsets;
  e->env_id_offset = env_id_offset;
#define A(f, T, cnt) e->f = (T*)or_zalloc(sizeof(T) * (size_t)(cnt))
  A(x, double, n); A(y, double, n); A(heading, double, n); A(vl, double, n); A(va, double, n);
  A(start_x, double, n); A(start_y, double, n); A(start_cos, double, n); A(start_sin, double, n);
  A(pk, double, n); A(pdt, double, n); A(pvl, double, n); A(pva, double, n); A(psig, double, n);
  A(pdelay, int64_t, n); A(step_count, int64_t, n); A(needs_reset, uint8_t, n);
  A(last_scan, double, n * n_beams); A(qv, double, n * (OR_MAX_DELAY + 1) * 2);
  A(qhead, int32_t, n); A(qlen, int32_t, n); A(rng, OrStream, n);
  A(ep_return, double, n); A(episodes, int64_t, n); A(arrivals, int64_t, n);
  A(return_sum, double, n); A(first_event, int8_t, n); A(first_return, double, n);
  A(first_steps, int64_t, n); A(scan_raw, double, n * n_beams); A(scan_min, double, n);
  A(cells_last, int64_t, n * n_beams); A(cells_store, int64_t, n * n_beams);
#undef A
  for (int64_t i = 0; i < n; ++i) { e->needs_reset[i] = 1; e->first_event[i] = -1; }
  return e;
}

void or_env_destroy(OrEnv* e) {
  if (!e) return;
  void* ptrs[] = {e->x, e->y, e->heading, e->vl, e->va, e->start_x, e->start_y, e->start_cos,
                  e->start_sin, e->pk, e->pdt, e->pvl, e->pva, e->psig, e->pdelay, e->step_count,
                  e->needs_reset, e->last_scan, e->qv, e->qhead, e->qlen, e->rng, e->ep_return,
                  e->episodes, e->arrivals, e->return_sum, e->first_event, e->first_return,
                  e->first_steps, e->scan_raw, e->scan_min, e->cells_last, e->cells_store};
  for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) free(ptrs[i]);
  free(e);
}

/* kinematics.py:17-19: pi - np.mod(pi - a, 2 pi); np.mod = fmod + sign fix */
static double or_wrap(double a) {
  const double two_pi = 2.0 * M_PI;
  double b = M_PI - a;
  double m = fmod(b, two_pi);
  if (m != 0.0) {
    if ((m < 0) != (two_pi < 0)) m += two_pi;
  } else {
    m = copysign(0.0, two_pi);
  }
  return M_PI - m;
}

/* reward.py:33-37 */
static double or_bearing(double x, double y, double h, double gx, double gy) {
  return or_wrap(atan2(gy - y, gx - x) - h);
}

/* reward.py:40-52 */
static double or_cross_track(double x, double y, double sx, double sy, double gx, double gy) {
  double vx = gx - sx, vy = gy - sy;
  double len2 = vx * vx + vy * vy;
  double safe = len2 > 0 ? len2 : 1.0;
  double t = ((x - sx) * vx + (y - sy) * vy) / safe;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  if (!(len2 > 0)) t = 0.0;
  double ex = x - (sx + t * vx), ey = y - (sy + t * vy);
  return sqrt(ex * ex + ey * ey);
}

static double or_clip(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* core.py:223-241 for one lane: scan at the current pose, then noise */
static void or_scan_lane(OrEnv* e, int64_t i) {
  int R = e->n_beams;
  int64_t m = e->map_index[i];
  const uint8_t* occ = e->occ + m * e->H * e->W;
  const double* edt = e->edt + m * e->H * e->W;
  double* raw = e->scan_raw + i * R;
  double mn = INFINITY;
  for (int j = 0; j < R; ++j) {
    double ang = e->heading[i] + e->offsets[j]; /* core.py:224 */
    raw[j] = or_cast_one(occ, edt, e->H, e->W, e->x[i], e->y[i], cos(ang), sin(ang), e->cell,
                         e->max_range, e->cells_last + i * R + j, NULL);
    if (raw[j] < mn) mn = raw[j];
  }
  e->scan_min[i] = mn; /* core.py:205 */
  double z[1024];
  or_normals(&e->rng[i], z, R); /* core.py:240: normal(0, sigma_i, R) */
  for (int j = 0; j < R; ++j)
    e->last_scan[i * R + j] = or_clip(raw[j] + (0.0 + e->psig[i] * z[j]), 0.0, e->max_range);
}

/* core.py:243-258 */
static void or_encode_lane(OrEnv* e, int64_t i, float* out) {
  int64_t m = e->map_index[i];
  double gx = e->goal_x[m], gy = e->goal_y[m];
  double rel_x = gx - e->x[i], rel_y = gy - e->y[i];
  double c0 = e->start_cos[i], s0 = e->start_sin[i], dist = e->plan_dist[m];
  double alpha = or_bearing(e->x[i], e->y[i], e->heading[i], gx, gy);
  out[0] = (float)((c0 * rel_x + s0 * rel_y) / dist);
  out[1] = (float)((-s0 * rel_x + c0 * rel_y) / dist);
  out[2] = (float)(alpha / M_PI);
  out[3] = (float)(e->vl[i] / e->pvl[i]);
  out[4] = (float)(e->va[i] / e->pva[i]);
  for (int j = 0; j < e->n_beams; ++j)
    out[5 + j] = (float)(e->last_scan[i * e->n_beams + j] / e->max_range);
}

/* core.py:114-161 (rng already bound to the lane) */
static int or_reset_lane(OrEnv* e, int64_t i, float* obs) {
  const double* rg = e->ranges + 12 * i;
  OrStream* s = &e->rng[i];
  /* DiversityRanges.sample, params.py:112-121 (draw order fixed) */
  e->pk[i] = or_uniform(s, rg[0], rg[1]);
  e->pdt[i] = or_uniform(s, rg[2], rg[3]);
  e->pdelay[i] = or_integers(s, (int64_t)rg[4], (int64_t)rg[5] + 1);
  e->pvl[i] = or_uniform(s, rg[6], rg[7]);
  e->pva[i] = or_uniform(s, rg[8], rg[9]);
  e->psig[i] = or_uniform(s, rg[10], rg[11]);
  int64_t m = e->map_index[i];
  const double* sp = e->spawn + 4 * m;
  const uint8_t* occ = e->occ + m * e->H * e->W;
  double sx = 0, sy = 0, sth = 0;
  int ok = 0;
  for (int a = 0; a < e->spawn_attempts; ++a) { /* core.py:135-147 */
    sx = or_uniform(s, sp[0], sp[2]);
    sy = or_uniform(s, sp[1], sp[3]);
    sth = or_uniform(s, -M_PI, M_PI);
    if (!or_disc_one(occ, e->H, e->W, sx, sy, e->robot_radius, e->cell)) { ok = 1; break; }
  }
  if (!ok) { e->err_lane = (int)i; return OR_EMAP; }
  e->x[i] = sx; e->y[i] = sy; e->heading[i] = sth; /* core.py:149-156 */
  e->start_x[i] = sx; e->start_y[i] = sy;
  e->start_cos[i] = cos(sth); e->start_sin[i] = sin(sth);
  e->vl[i] = 0.0; e->va[i] = 0.0;
  e->step_count[i] = 0;
  e->needs_reset[i] = 0;
  e->qhead[i] = 0; e->qlen[i] = (int32_t)e->pdelay[i];
  for (int q = 0; q < e->qlen[i]; ++q) {
    e->qv[(i * (OR_MAX_DELAY + 1) + q) * 2 + 0] = 0.0;
    e->qv[(i * (OR_MAX_DELAY + 1) + q) * 2 + 1] = 0.0;
  }
  or_scan_lane(e, i); /* core.py:158-161 */
  or_encode_lane(e, i, obs);
  return OR_OK;
}

/* vecenv.py:84-92 with the Philox stream contract instead of SeedSequence */
int or_env_reset_all(OrEnv* e, uint64_t seed, float* states) {
  int D = 5 + e->n_beams;
  e->seed = seed;
  for (int64_t i = 0; i < e->n; ++i) {
    OrStream s = {seed, (uint32_t)(e->env_id_offset + i), 0u, 0ull};
    e->rng[i] = s;
    int rc = or_reset_lane(e, i, states + i * D);
    if (rc) return rc;
    e->ep_return[i] = 0.0;
    e->first_event[i] = -1;
  }
  return OR_OK;
}

/* SimBatch.step_all (core.py:165-219) + VecEnv.step_batch (vecenv.py:94-116).
 * Outputs: states (post-reset), store_states (pre-reset s'), rewards (f64),
 * dones, truncated, events. */
int or_env_step(OrEnv* e, const int64_t* actions, float* states, float* store_states,
                double* rewards, uint8_t* dones, uint8_t* truncated, int8_t* events) {
  int64_t n = e->n;
  int R = e->n_beams, D = 5 + R;
  for (int64_t i = 0; i < n; ++i) /* core.py:169-170 */
    if (actions[i] < 0 || actions[i] >= e->n_actions) return OR_EACTION;
  for (int64_t i = 0; i < n; ++i) /* core.py:171-174 */
    if (e->needs_reset[i]) { e->err_lane = (int)i; return OR_EEPISODE; }
  for (int64_t i = 0; i < n; ++i) {
    int64_t m = e->map_index[i];
    /* delay queue: append target, pop oldest (core.py:176-182) */
    double* q = e->qv + i * (OR_MAX_DELAY + 1) * 2;
    int cap = OR_MAX_DELAY + 1;
    int tail = (e->qhead[i] + e->qlen[i]) % cap;
    q[tail * 2 + 0] = e->action_table[actions[i]][0];
    q[tail * 2 + 1] = e->action_table[actions[i]][1];
    double mv = q[e->qhead[i] * 2 + 0], mw = q[e->qhead[i] * 2 + 1];
    e->qhead[i] = (e->qhead[i] + 1) % cap;
    /* apply_kinematics, kinematics.py:22-36 */
    double k = e->pk[i];
    double v0 = k * e->vl[i] + (1.0 - k) * mv;
    double v1 = k * e->va[i] + (1.0 - k) * mw;
    v0 = fmin(fmax(v0, -e->pvl[i]), e->pvl[i]);
    v1 = fmin(fmax(v1, -e->pva[i]), e->pva[i]);
    e->vl[i] = v0; e->va[i] = v1;
    /* integrate_unicycle, kinematics.py:39-63 */
    double h = e->heading[i], dt = e->pdt[i];
    double sin0 = sin(h), cos0 = cos(h);
    double h1 = h + v1 * dt;
    double sin1 = sin(h1), cos1 = cos(h1);
    int curved = fabs(v1) >= 1e-6;
    double omega = curved ? v1 : 1.0;
    double radius = v0 / omega;
    double ddx = curved ? radius * (sin1 - sin0) : v0 * cos0 * dt;
    double ddy = curved ? -radius * (cos1 - cos0) : v0 * sin0 * dt;
    e->x[i] = e->x[i] + ddx;
    e->y[i] = e->y[i] + ddy;
    e->heading[i] = or_wrap(h1);
    /* events, core.py:189-201 */
    const uint8_t* occ = e->occ + m * e->H * e->W;
    int coll = or_disc_one(occ, e->H, e->W, e->x[i], e->y[i], e->robot_radius, e->cell);
    double gdx = e->goal_x[m] - e->x[i], gdy = e->goal_y[m] - e->y[i];
    double d1 = sqrt(gdx * gdx + gdy * gdy);
    int arrived = !coll && d1 <= e->goal_r[m];
    e->step_count[i] += 1;
    int timed_out = !coll && !arrived && e->step_count[i] >= e->timeout_steps;
    int8_t ev = coll ? 1 : (arrived ? 2 : (timed_out ? 3 : 0));
    /* scan + noise (core.py:203-206) */
    or_scan_lane(e, i);
    memcpy(e->cells_store + i * R, e->cells_last + i * R, sizeof(int64_t) * (size_t)R);
    /* reward, reward.py:55-83 */
    double alpha = or_bearing(e->x[i], e->y[i], e->heading[i], e->goal_x[m], e->goal_y[m]);
    double d2 = or_cross_track(e->x[i], e->y[i], e->start_x[i], e->start_y[i], e->goal_x[m],
                               e->goal_y[m]);
    double D_ = e->plan_dist[m];
    double rew;
    if (ev == 1) rew = -10.0;
    else if (ev == 2) rew = 75.0;
    else {
      double r_d1 = or_clip(1.0 - d1 / D_, 0.0, 1.0);
      double r_d2 = or_clip(1.0 - d2 / D_, 0.0, 1.0);
      double r_v = v0 > e->pvl[i] / 2.0 ? 1.0 : 0.0;
      double r_a = or_clip(1.0 - 2.0 * fabs(alpha) / M_PI, -1.0, 1.0);
      double r_p = e->scan_min[i] < e->proximity ? -1.0 : 0.0;
      rew = 0.3 * r_d1 + 0.1 * r_d2 + 0.3 * r_v + 0.3 * r_a + 0.1 * r_p;
    }
    rewards[i] = rew;
    dones[i] = (uint8_t)(coll || arrived); /* core.py:216-217 */
    truncated[i] = (uint8_t)timed_out;
    events[i] = ev;
    if (coll || arrived || timed_out) e->needs_reset[i] = 1;
    or_encode_lane(e, i, store_states + i * D);
    memcpy(states + i * D, store_states + i * D, sizeof(float) * (size_t)D);
  }
  /* VecEnv bookkeeping + auto-reset, vecenv.py:96-114 */
  for (int64_t i = 0; i < n; ++i) e->ep_return[i] += rewards[i];
  for (int64_t i = 0; i < n; ++i) {
    if (!(dones[i] || truncated[i])) continue;
    double ret = e->ep_return[i];
    e->episodes[i] += 1;
    e->return_sum[i] += ret;
    if (events[i] == 2) e->arrivals[i] += 1;
    e->recent[e->recent_count % 256] = ret;
    e->recent_count += 1;
    if (e->first_event[i] < 0) {
      e->first_event[i] = events[i];
      e->first_return[i] = ret;
      e->first_steps[i] = e->step_count[i];
    }
    e->ep_return[i] = 0.0;
    if (e->auto_reset) {
      int rc = or_reset_lane(e, i, states + i * D);
      if (rc) return rc;
    }
  }
  return OR_OK;
}

/* read-only views for tests */
void or_env_get_pose(const OrEnv* e, double* x, double* y, double* h, double* vl, double* va,
                     int64_t* step_count, uint64_t* ctr) {
  for (int64_t i = 0; i < e->n; ++i) {
    x[i] = e->x[i]; y[i] = e->y[i]; h[i] = e->heading[i]; vl[i] = e->vl[i]; va[i] = e->va[i];
    step_count[i] = e->step_count[i]; ctr[i] = e->rng[i].ctr;
  }
}

void or_env_get_stats(const OrEnv* e, int64_t* episodes, int64_t* arrivals, double* return_sum,
                      int8_t* first_event, double* first_return, int64_t* first_steps,
                      double* recent, int64_t* recent_count) {
  for (int64_t i = 0; i < e->n; ++i) {
    episodes[i] = e->episodes[i]; arrivals[i] = e->arrivals[i]; return_sum[i] = e->return_sum[i];
    first_event[i] = e->first_event[i]; first_return[i] = e->first_return[i];
    first_steps[i] = e->first_steps[i];
  }
  memcpy(recent, e->recent, sizeof(e->recent));
  *recent_count = e->recent_count;
}

void or_env_reset_stats(OrEnv* e) {
  for (int64_t i = 0; i < e->n; ++i) { e->episodes[i] = 0; e->arrivals[i] = 0; e->return_sum[i] = 0; }
  e->recent_count = 0;
}

int or_env_err_lane(const OrEnv* e) { return e->err_lane; }

/* hit cells of the last step's post-step scans and of the scans behind the
 * current states rows, plus last_scan (core.py:97), n * n_beams each */
void or_env_get_cells(const OrEnv* e, int64_t* store, int64_t* last, double* last_scan) {
  const size_t k = (size_t)e->n * (size_t)e->n_beams;
  if (store) memcpy(store, e->cells_store, sizeof(int64_t) * k);
  if (last) memcpy(last, e->cells_last, sizeof(int64_t) * k);
  if (last_scan) memcpy(last_scan, e->last_scan, sizeof(double) * k);
}
