// sp_env.cu -- the fused Sparrow step (+auto-reset) kernel for sm_100a.
//
// One launch per VecEnv.step_batch (vecenv.py:94-116 -> core.py:165-219, with
// the auto-reset of core.py:114-161 fused in).  Layout and schedule:
//
// * Lanes (env copies) are stored struct-of-arrays in MAP-MAJOR slot order;
//   env_of_slot maps a slot back to the caller's row (outputs keep the
//   reference row order).  Each CTA owns a contiguous slot range, so it needs
//   one map (rarely two) at a time.
// * Per map, two tables live in shared memory, staged by one TMA bulk copy
//   (cp.async.bulk + mbarrier): a 1-bit occupancy bitmap (H x ceil(W/32) u32)
//   and a 2x2-block "free box" table (u8: 0 = block holds an occupied cell,
//   else 1 + r where the (2r+1)^2 blocks around it are all free).  366 x 366
//   cells -> 17.6 KB + 33.5 KB.
// * A warp takes a batch of E lanes.  Env math runs lane-per-env in fp64 with
//   the reference's rounding order; LiDAR rays run from a per-warp ray queue
//   (lane-per-ray, idle lanes refill by ballot) so divergent ray lengths do
//   not idle the warp.  Noise is drawn lane-per-env into the staging row.
// * The march visits the same cells as the reference DDA (_cy.pyx:89-105) but
//   jumps over free boxes in one step: at cell (ix,iy) with free box B, the
//   ray leaves B through the face with the smaller exit parameter (ties go to
//   x, as tmx <= tmy does), re-entering the cell grid at the cell containing
//   the exit point (clamped into B's span on the other axis).  Only free cells
//   are skipped, so the first occupied cell is the reference's (up to
//   exact-corner rounding, the same ambiguity the reference's own EDT jump
//   has, _cy.pyx:62-88).
#include "sp_env.cuh"

namespace sp {

// ------------------------------------------------------------ TMA helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------- map view ---
struct MapView {
  const uint8_t* blk;
  const uint32_t* bits;
  int W, H, Wb, WW;
  __device__ __forceinline__ uint32_t code(int ix, int iy) const {
    return blk[(iy >> 1) * Wb + (ix >> 1)];
  }
  __device__ __forceinline__ bool occ(int ix, int iy) const {
    return (bits[iy * WW + (ix >> 5)] >> (ix & 31)) & 1u;
  }
};

// disc_collides for one disc (_cy.pyx:109-158), exact fp64 test; the block
// table proves most discs free with one lookup.
__device__ __forceinline__ bool disc_hits(const MapView& mv, const EnvDev& d, double x, double y) {
  const double r = d.radius, cell = d.cell;
  if (x - r < 0.0 || y - r < 0.0 || x + r > (double)d.W * cell || y + r > (double)d.H * cell)
    return true;  // :124-126
  int cx = (int)floor(x * d.inv_cell), cy = (int)floor(y * d.inv_cell);
  if (cx >= 0 && cx < d.W && cy >= 0 && cy < d.H) {
    uint32_t c = mv.code(cx, cy);
    if (c > (uint32_t)d.need_r) return false;  // free box covers the whole bbox
  }
  int ix0 = (int)floor(ddiv(dsub(x, r), cell)); if (ix0 < 0) ix0 = 0;  // :128-135
  int ix1 = (int)floor(ddiv(dadd(x, r), cell)); if (ix1 > d.W - 1) ix1 = d.W - 1;
  int iy0 = (int)floor(ddiv(dsub(y, r), cell)); if (iy0 < 0) iy0 = 0;
  int iy1 = (int)floor(ddiv(dadd(y, r), cell)); if (iy1 > d.H - 1) iy1 = d.H - 1;
  const double r2 = dmul(r, r);
  for (int iy = iy0; iy <= iy1; ++iy) {
    const uint32_t* rowp = mv.bits + iy * mv.WW;
    for (int w = ix0 >> 5; w <= (ix1 >> 5); ++w) {
      uint32_t m = rowp[w];
      int lo = w << 5;
      if (ix0 > lo) m &= ~0u << (ix0 - lo);
      if (ix1 - lo < 31) m &= (2u << (ix1 - lo)) - 1u;
      while (m) {
        int ix = lo + __ffs(m) - 1;
        m &= m - 1;
        double clo = dmul((double)ix, cell), chi = dadd(clo, cell);  // :141-153
        double nx = x > clo ? x : clo;
        if (nx > chi) nx = chi;
        double rlo = dmul((double)iy, cell), rhi = dadd(rlo, cell);
        double ny = y > rlo ? y : rlo;
        if (ny > rhi) ny = rhi;
        double ddx = dsub(x, nx), ddy = dsub(y, ny);
        if (dadd(dmul(ddx, ddx), dmul(ddy, ddy)) <= r2) return true;
      }
    }
  }
  return false;
}

// ---------------------------------------------------------------- rays ---
struct Ray {
  double x0, y0, dx, dy, idx, idy, t;
  int ix, iy;
};

// One free-box step.  Returns true when the ray is finished (r.t = range).
__device__ __forceinline__ bool ray_step(Ray& r, const MapView& mv, const EnvDev& d, int& hit) {
  uint32_t code = mv.code(r.ix, r.iy);
  int lox, hix, loy, hiy;
  if (code == 0u) {
    if (mv.occ(r.ix, r.iy)) {  // entered an occupied cell at r.t (<= max_range)
      hit = r.iy * d.W + r.ix;
      return true;
    }
    lox = hix = r.ix;
    loy = hiy = r.iy;
  } else {
    int rr = (int)code - 1;
    int bx = r.ix >> 1, by = r.iy >> 1;
    lox = (bx - rr) << 1;
    hix = ((bx + rr) << 1) + 1;
    loy = (by - rr) << 1;
    hiy = ((by + rr) << 1) + 1;
  }
  const bool px = r.dx >= 0.0, py = r.dy >= 0.0;
  const double X = (double)(px ? hix + 1 : lox), Y = (double)(py ? hiy + 1 : loy);
  const double tx = (X * d.cell - r.x0) * r.idx;
  const double ty = (Y * d.cell - r.y0) * r.idy;
  if (tx <= ty) {  // leave through the x face (tie -> x, as _cy.pyx:89)
    r.t = tx;
    r.ix = px ? hix + 1 : lox - 1;
    if (code != 0u) {
      int c = (int)floor((r.y0 + tx * r.dy) * d.inv_cell);
      r.iy = min(max(c, loy), hiy);
    }
  } else {
    r.t = ty;
    r.iy = py ? hiy + 1 : loy - 1;
    if (code != 0u) {
      int c = (int)floor((r.x0 + ty * r.dx) * d.inv_cell);
      r.ix = min(max(c, lox), hix);
    }
  }
  if (r.t > d.max_range) {  // :97-99
    r.t = d.max_range;
    hit = -1;
    return true;
  }
  if ((unsigned)r.ix >= (unsigned)d.W || (unsigned)r.iy >= (unsigned)d.H) {  // :100-102
    hit = -1;
    return true;
  }
  return false;
}

// Returns true if finished during setup (origin outside the grid -> 0).
__device__ __forceinline__ bool ray_setup(Ray& r, double x0, double y0, double ch, double sh,
                                          double2 cs, const EnvDev& d, int& hit) {
  r.x0 = x0;
  r.y0 = y0;
  r.dx = ch * cs.x - sh * cs.y;  // cos(h + o_j)
  r.dy = sh * cs.x + ch * cs.y;  // sin(h + o_j)
  r.idx = r.dx != 0.0 ? 1.0 / r.dx : __longlong_as_double(0x7ff0000000000000ll);
  r.idy = r.dy != 0.0 ? 1.0 / r.dy : __longlong_as_double(0x7ff0000000000000ll);
  r.t = 0.0;
  r.ix = (int)floor(x0 * d.inv_cell);
  r.iy = (int)floor(y0 * d.inv_cell);
  if ((unsigned)r.ix >= (unsigned)d.W || (unsigned)r.iy >= (unsigned)d.H) {  // :37-39
    hit = -1;
    return true;
  }
  return false;
}

// Per-warp scratch (shared memory).
struct WarpSmem {
  double *px, *py, *ch, *sh, *sig;
  unsigned long long* smin;
  int32_t* list;  // batch-local env index per queue entry
  float* stage;   // E x D staging rows
};

__device__ __forceinline__ WarpSmem warp_smem(uint8_t* base, int D) {
  WarpSmem w;
  w.px = (double*)base;
  w.py = w.px + 32;
  w.ch = w.py + 32;
  w.sh = w.ch + 32;
  w.sig = w.sh + 32;
  w.smin = (unsigned long long*)(w.sig + 32);
  w.list = (int32_t*)(w.smin + 32);
  w.stage = (float*)(w.list + 32);
  (void)D;
  return w;
}

// Ray queue over n_env envs (ws.list) x R beams.  fin(e, j, t, hit).
template <bool kHit, class Fin>
__device__ __forceinline__ void ray_phase(const MapView& mv, const EnvDev& d, const WarpSmem& ws,
                                          const double2* beam, int n_env, Fin fin) {
  const int R = d.R;
  const int total = n_env * R;
  int next = 0;
  bool active = false;
  int e = 0, j = 0;
  Ray r;
  for (;;) {
    const unsigned need = __ballot_sync(SP_FULL, !active);
    if (need != 0u && next < total) {
      const int my = next + __popc(need & lanemask_lt());
      next += __popc(need);
      if (!active && my < total) {
        e = ws.list[my / R];
        j = my - (my / R) * R;
        int hit;
        if (ray_setup(r, ws.px[e], ws.py[e], ws.ch[e], ws.sh[e], beam[j], d, hit)) {
          fin(e, j, 0.0, hit);
        } else {
          active = true;
        }
      }
    }
    if (!__any_sync(SP_FULL, active)) {
      if (next >= total) break;
      continue;
    }
    if (active) {
      int hit;
      if (ray_step(r, mv, d, hit)) {
        fin(e, j, r.t, kHit ? hit : -1);
        active = false;
      }
    }
  }
}

__device__ __forceinline__ void set_error(const EnvDev& d, int code, int64_t row) {
  if (atomicCAS(d.err, 0, code) == 0) d.err[1] = (int32_t)row;
}

// Fill stage[5 .. 5+R) of one row with standard normals (core.py:240 draws).
__device__ __forceinline__ void draw_noise_row(const EnvDev& d, uint32_t gid, uint64_t& ctr,
                                               float* row) {
  const int R = d.R;
  for (int j = 0; j < R; j += 4) {
    Block4 b = stream_block(d.seed, gid, 0u, ctr++);
    float z[4];
    draw_normals4(b, z);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j + u < R) row[5 + j + u] = z[u];
  }
}

// reward.py:33-37
__device__ __forceinline__ double bearing_error(double x, double y, double h, double gx,
                                                double gy) {
  return wrap_angle(dsub(atan2(dsub(gy, y), dsub(gx, x)), h));
}

// reward.py:40-52
__device__ __forceinline__ double cross_track(double x, double y, double sx, double sy, double gx,
                                              double gy) {
  double vx = dsub(gx, sx), vy = dsub(gy, sy);
  double len2 = dadd(dmul(vx, vx), dmul(vy, vy));
  double safe = len2 > 0.0 ? len2 : 1.0;
  double t = dclip(ddiv(dadd(dmul(dsub(x, sx), vx), dmul(dsub(y, sy), vy)), safe), 0.0, 1.0);
  if (!(len2 > 0.0)) t = 0.0;
  double ex = dsub(x, dadd(sx, dmul(t, vx))), ey = dsub(y, dadd(sy, dmul(t, vy)));
  return __dsqrt_rn(dadd(dmul(ex, ex), dmul(ey, ey)));
}

// Lane state carried through one warp batch.
struct Lane {
  double x, y, h, vl, va, ret, sx, sy, c0, s0, k, dt, vml, vma, sig;
  uint64_t hist0, ctr;
  int32_t step, delay;
};

__device__ __forceinline__ void header_row(const EnvDev& d, const MapConst& mc, const Lane& L,
                                           float* row) {
  // core.py:243-258 (columns 0..4; LiDAR columns are written by the ray phase)
  double rx = dsub(mc.goal_x, L.x), ry = dsub(mc.goal_y, L.y);
  double alpha = bearing_error(L.x, L.y, L.h, mc.goal_x, mc.goal_y);
  row[0] = (float)ddiv(dadd(dmul(L.c0, rx), dmul(L.s0, ry)), mc.plan_dist);
  row[1] = (float)ddiv(dadd(dmul(-L.s0, rx), dmul(L.c0, ry)), mc.plan_dist);
  row[2] = (float)ddiv(alpha, SP_PI);
  row[3] = (float)ddiv(L.vl, L.vml);
  row[4] = (float)ddiv(L.va, L.vma);
}

// core.py:114-156 for one lane (stream already bound).  false = no spawn.
__device__ __forceinline__ bool reset_lane(const EnvDev& d, const MapView& mv, const MapConst& mc,
                                           int64_t s, uint32_t gid, Lane& L) {
  const double* rg = d.ranges + (d.ranges_shared ? 0 : 12 * s);
  // DiversityRanges.sample (params.py:112-121): U U I U U U
  L.k = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), rg[0], rg[1]);
  L.dt = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), rg[2], rg[3]);
  L.delay = (int32_t)draw_integer(stream_block(d.seed, gid, 0u, L.ctr++), (int64_t)rg[4],
                                  (int64_t)rg[5] + 1);
  L.vml = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), rg[6], rg[7]);
  L.vma = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), rg[8], rg[9]);
  L.sig = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), rg[10], rg[11]);
  // spawn rejection (core.py:135-147)
  bool ok = false;
  double x = 0, y = 0, th = 0;
  for (int a = 0; a < d.spawn_attempts; ++a) {
    x = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), mc.spawn[0], mc.spawn[2]);
    y = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), mc.spawn[1], mc.spawn[3]);
    th = draw_uniform(stream_block(d.seed, gid, 0u, L.ctr++), -SP_PI, SP_PI);
    if (!disc_hits(mv, d, x, y)) {
      ok = true;
      break;
    }
  }
  if (!ok) return false;
  L.x = x; L.y = y; L.h = th;  // core.py:149-156
  L.sx = x; L.sy = y;
  L.c0 = cos(th);
  L.s0 = sin(th);
  L.vl = 0.0; L.va = 0.0;
  L.step = 0;
  L.hist0 = ~0ull;  // d x (0, 0): 4-bit code 15 everywhere
  return true;
}

// ------------------------------------------------------------ the batch ---
__device__ __noinline__ void env_batch(const EnvDev& d, const StepArgs& a, const MapView& mv,
                                       const MapConst& mc, const double2* beam, const WarpSmem& ws,
                                       int64_t s0, int E, int lane) {
  const int D = d.D;
  const bool act = lane < E;
  const int64_t s = s0 + lane;
  const int64_t row = act ? d.env_of_slot[s] : 0;
  const uint32_t gid = (uint32_t)(d.env_id_offset + row);
  float* my_stage = ws.stage + lane * D;
  Lane L;
  bool live = false;  // this lane takes part in the step
  bool ended = false;
  int8_t ev = 0;
  bool coll = false, arrived = false, timed_out = false;
  double d1 = 0.0;

  if (act) {
    L.x = d.x[s]; L.y = d.y[s]; L.h = d.h[s]; L.vl = d.vl[s]; L.va = d.va[s]; L.ret = d.ret[s];
    L.sx = d.sx[s]; L.sy = d.sy[s]; L.c0 = d.c0[s]; L.s0 = d.s0[s];
    L.k = d.pk[s]; L.dt = d.pdt[s]; L.vml = d.pvl[s]; L.vma = d.pva[s]; L.sig = d.psig[s];
    L.ctr = d.ctr[s]; L.step = d.step[s]; L.delay = d.delay[s];
    L.hist0 = L.delay > 0 ? d.hist[s] : 0ull;
    ws.list[lane] = lane;
  }
  if (a.mode == MODE_STEP && act) {
    const int64_t av = a.actions[row];
    if (av < 0 || av >= d.n_actions) {
      set_error(d, SP_EACTION, row);
    } else if (d.needs_reset[s]) {
      set_error(d, SP_EEPISODE, row);
    } else {
      live = true;
      // delay queue (core.py:176-182): matured = action from `delay` steps ago
      uint32_t code;
      if (L.delay == 0) {
        code = (uint32_t)av;
      } else {
        const int q = L.delay - 1;
        uint64_t w = q < 16 ? L.hist0 : d.hist[(int64_t)(q >> 4) * d.n + s];
        code = (uint32_t)(w >> (4 * (q & 15))) & 15u;
        // push av: shift the 4-bit history by one entry across the used words
        const int nw = (L.delay + 15) >> 4;
        uint64_t carry = (uint64_t)av;
        for (int wi = 0; wi < nw; ++wi) {
          uint64_t cur = wi == 0 ? L.hist0 : d.hist[(int64_t)wi * d.n + s];
          uint64_t nxt = (cur << 4) | carry;
          carry = cur >> 60;
          if (wi == 0) L.hist0 = nxt;
          else d.hist[(int64_t)wi * d.n + s] = nxt;
        }
      }
      const double mv_ = d.action_v[code], mw_ = d.action_w[code];
      // apply_kinematics (kinematics.py:22-36)
      double v0 = dadd(dmul(L.k, L.vl), dmul(dsub(1.0, L.k), mv_));
      double v1 = dadd(dmul(L.k, L.va), dmul(dsub(1.0, L.k), mw_));
      v0 = dclip(v0, -L.vml, L.vml);
      v1 = dclip(v1, -L.vma, L.vma);
      L.vl = v0; L.va = v1;
      // integrate_unicycle (kinematics.py:39-63)
      double sin0, cos0, sin1, cos1;
      sincos(L.h, &sin0, &cos0);
      const double h1 = dadd(L.h, dmul(v1, L.dt));
      sincos(h1, &sin1, &cos1);
      double ddx, ddy;
      if (fabs(v1) >= 1e-6) {
        const double radius = ddiv(v0, v1);
        ddx = dmul(radius, dsub(sin1, sin0));
        ddy = dmul(-radius, dsub(cos1, cos0));
      } else {
        ddx = dmul(dmul(v0, cos0), L.dt);
        ddy = dmul(dmul(v0, sin0), L.dt);
      }
      L.x = dadd(L.x, ddx);
      L.y = dadd(L.y, ddy);
      L.h = wrap_angle(h1);
      // events (core.py:189-201)
      coll = disc_hits(mv, d, L.x, L.y);
      const double gdx = dsub(mc.goal_x, L.x), gdy = dsub(mc.goal_y, L.y);
      d1 = __dsqrt_rn(dadd(dmul(gdx, gdx), dmul(gdy, gdy)));
      arrived = !coll && d1 <= mc.goal_r;
      L.step += 1;
      timed_out = !coll && !arrived && L.step >= d.timeout;
      ev = coll ? 1 : (arrived ? 2 : (timed_out ? 3 : 0));
      ended = coll || arrived || timed_out;
      // noise for this step's scan (core.py:237-241), staged as z
      draw_noise_row(d, gid, L.ctr, my_stage);
      double sh_, ch_;
      sincos(L.h, &sh_, &ch_);
      ws.px[lane] = L.x; ws.py[lane] = L.y; ws.ch[lane] = ch_; ws.sh[lane] = sh_;
      ws.sig[lane] = L.sig;
      ws.smin[lane] = 0x7ff0000000000000ull;  // +inf
    }
  }

  const double max_range = d.max_range;
  auto fin_obs = [&](int e, int j, double t, int) {
    float* rowp = ws.stage + e * D;
    const double z = (double)rowp[5 + j];
    const double v = dclip(dadd(t, dadd(0.0, dmul(ws.sig[e], z))), 0.0, max_range);
    rowp[5 + j] = (float)ddiv(v, max_range);
    atomicMin(&ws.smin[e], (unsigned long long)__double_as_longlong(t + 0.0));
  };

  if (a.mode == MODE_STEP) {
    const unsigned live_mask = __ballot_sync(SP_FULL, live);
    // compact the live lanes into the queue list
    if (live) ws.list[__popc(live_mask & lanemask_lt())] = lane;
    __syncwarp();
    ray_phase<false>(mv, d, ws, beam, __popc(live_mask), fin_obs);
    __syncwarp();
    if (live) {
      const double smin = __longlong_as_double((long long)ws.smin[lane]);
      // reward (reward.py:55-83)
      double rew;
      if (ev == 1) {
        rew = -10.0;
      } else if (ev == 2) {
        rew = 75.0;
      } else {
        const double alpha = bearing_error(L.x, L.y, L.h, mc.goal_x, mc.goal_y);
        const double d2 = cross_track(L.x, L.y, L.sx, L.sy, mc.goal_x, mc.goal_y);
        const double r_d1 = dclip(dsub(1.0, ddiv(d1, mc.plan_dist)), 0.0, 1.0);
        const double r_d2 = dclip(dsub(1.0, ddiv(d2, mc.plan_dist)), 0.0, 1.0);
        const double r_v = L.vl > ddiv(L.vml, 2.0) ? 1.0 : 0.0;
        const double r_a = dclip(dsub(1.0, ddiv(dmul(2.0, fabs(alpha)), SP_PI)), -1.0, 1.0);
        const double r_p = smin < d.proximity ? -1.0 : 0.0;
        rew = dadd(dadd(dadd(dadd(dmul(0.3, r_d1), dmul(0.1, r_d2)), dmul(0.3, r_v)),
                        dmul(0.3, r_a)),
                   dmul(0.1, r_p));
      }
      header_row(d, mc, L, my_stage);
      a.rewards[row] = rew;
      a.dones[row] = (uint8_t)(coll || arrived);
      a.truncated[row] = (uint8_t)timed_out;
      a.events[row] = ev;
      // VecEnv bookkeeping (vecenv.py:96-112)
      L.ret = dadd(L.ret, rew);
      if (ended) {
        d.episodes[s] += 1;
        d.return_sum[s] = dadd(d.return_sum[s], L.ret);
        if (ev == 2) d.arrivals[s] += 1;
        const unsigned long long k = atomicAdd(d.rec_count, 1ull);
        const uint64_t slot = k % d.rec_cap;
        d.rec_ret[slot] = L.ret;
        d.rec_key[slot] = (a.step_index << 32) | (uint64_t)row;
        if (d.first_event[s] < 0) {
          d.first_event[s] = ev;
          d.first_ret[s] = L.ret;
          d.first_steps[s] = L.step;
        }
        L.ret = 0.0;
      }
    }
    __syncwarp();
    // write s' rows (store_states) and, for lanes that keep running, states
    const unsigned live_mask2 = __ballot_sync(SP_FULL, live);
    const unsigned end_mask = __ballot_sync(SP_FULL, live && ended);
    for (int e = 0; e < E; ++e) {
      if (!((live_mask2 >> e) & 1u)) continue;
      const int64_t rr = d.env_of_slot[s0 + e];
      const float* src = ws.stage + e * D;
      const bool keep = !((end_mask >> e) & 1u) || !d.auto_reset;
      for (int c = lane; c < D; c += 32) {
        const float v = src[c];
        a.store_states[rr * D + c] = v;
        if (keep) a.states[rr * D + c] = v;
      }
    }
    __syncwarp();
  }

  // ---- resets: auto-reset of ended lanes, or reset_all ------------------
  bool do_reset = (a.mode == MODE_RESET_ALL) ? act : (live && ended && d.auto_reset);
  bool spawned = false;
  if (do_reset) {
    spawned = reset_lane(d, mv, mc, s, gid, L);
    if (!spawned) set_error(d, SP_EMAP, row);
  }
  const unsigned reset_mask = __ballot_sync(SP_FULL, spawned);
  if (reset_mask != 0u) {
    if (spawned) {
      draw_noise_row(d, gid, L.ctr, my_stage);  // core.py:159-160
      ws.px[lane] = L.x; ws.py[lane] = L.y; ws.ch[lane] = L.c0; ws.sh[lane] = L.s0;
      ws.sig[lane] = L.sig;
      ws.smin[lane] = 0x7ff0000000000000ull;
      ws.list[__popc(reset_mask & lanemask_lt())] = lane;
    }
    __syncwarp();
    ray_phase<false>(mv, d, ws, beam, __popc(reset_mask), fin_obs);
    __syncwarp();
    if (spawned) header_row(d, mc, L, my_stage);
    __syncwarp();
    for (int e = 0; e < E; ++e) {
      if (!((reset_mask >> e) & 1u)) continue;
      const int64_t rr = d.env_of_slot[s0 + e];
      const float* src = ws.stage + e * D;
      for (int c = lane; c < D; c += 32) a.states[rr * D + c] = src[c];
    }
    __syncwarp();
  }

  // ---- write back the SoA state --------------------------------------------
  if (live || spawned) {
    d.x[s] = L.x; d.y[s] = L.y; d.h[s] = L.h; d.vl[s] = L.vl; d.va[s] = L.va;
    d.ret[s] = (a.mode == MODE_RESET_ALL) ? 0.0 : L.ret;
    d.ctr[s] = L.ctr;
    d.step[s] = L.step;
    if (L.delay > 0) d.hist[s] = L.hist0;
    d.needs_reset[s] = (uint8_t)(spawned ? 0 : (ended ? 1 : 0));
    if (spawned) {
      d.sx[s] = L.sx; d.sy[s] = L.sy; d.c0[s] = L.c0; d.s0[s] = L.s0;
      d.pk[s] = L.k; d.pdt[s] = L.dt; d.pvl[s] = L.vml; d.pva[s] = L.vma; d.psig[s] = L.sig;
      d.delay[s] = L.delay;
      for (int wi = 1; wi < ((L.delay + 15) >> 4); ++wi) d.hist[(int64_t)wi * d.n + s] = ~0ull;
      if (a.mode == MODE_RESET_ALL) d.first_event[s] = -1;
    }
  } else if (do_reset && !spawned && act) {
    d.ctr[s] = L.ctr;
  }
}

// Load map m's tables (TMA bulk copy into shared memory) -- or point at HBM.
__device__ __forceinline__ MapView bind_map(const EnvDev& d, int m, uint8_t* smem_maps,
                                            uint64_t* bar, uint32_t& phase) {
  const uint8_t* src = d.maps + (size_t)m * d.map_bytes;
  MapView mv;
  mv.W = d.W;
  mv.H = d.H;
  mv.Wb = d.Wb;
  mv.WW = d.WW;
  if (d.smem_maps) {
    __syncthreads();  // everyone is done with the previous map
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, d.map_bytes);
      tma_bulk_g2s(smem_maps, src, d.map_bytes, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    mv.blk = smem_maps;
    mv.bits = (const uint32_t*)(smem_maps + d.blk_bytes);
  } else {
    mv.blk = src;
    mv.bits = (const uint32_t*)(src + d.blk_bytes);
  }
  return mv;
}

__global__ void __launch_bounds__(768, 1) env_step_kernel(const __grid_constant__ EnvDev d, const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double2* beam = (double2*)(smem + d.off_beam);
  uint64_t* bar = (uint64_t*)(smem + d.off_bar);
  for (int j = threadIdx.x; j < d.R; j += blockDim.x) beam[j] = d.beam_cs[j];
  if (threadIdx.x == 0 && d.smem_maps) mbar_init(bar, 1);
  __syncthreads();
  const WarpSmem ws = warp_smem(smem + d.off_warps + (size_t)warp * d.warp_smem, d.D);
  uint32_t phase = 0;
  const int64_t sb = (int64_t)blockIdx.x * d.n / gridDim.x;
  const int64_t se = (int64_t)(blockIdx.x + 1) * d.n / gridDim.x;
  int64_t s = sb;
  int m = 0;
  while (s < se) {
    while (d.map_off[m + 1] <= s) ++m;
    const int64_t seg_end = min(se, d.map_off[m + 1]);
    const MapView mv = bind_map(d, m, smem, bar, phase);
    const MapConst mc = d.mconst[m];
    const int64_t nb = (seg_end - s + d.E - 1) / d.E;
    for (int64_t b = warp; b < nb; b += nwarps) {
      const int64_t s0 = s + b * d.E;
      const int E = (int)min((int64_t)d.E, seg_end - s0);
      env_batch(d, a, mv, mc, beam, ws, s0, E, lane);
    }
    s = seg_end;
  }
}

// Standalone LiDAR scan on caller poses (cfg4): the same marcher, no noise.
__global__ void __launch_bounds__(768, 1) env_scan_kernel(const __grid_constant__ EnvDev d, const __grid_constant__ ScanArgs q) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double2* beam = (double2*)(smem + d.off_beam);
  uint64_t* bar = (uint64_t*)(smem + d.off_bar);
  for (int j = threadIdx.x; j < d.R; j += blockDim.x) beam[j] = d.beam_cs[j];
  if (threadIdx.x == 0 && d.smem_maps) mbar_init(bar, 1);
  __syncthreads();
  const WarpSmem ws = warp_smem(smem + d.off_warps + (size_t)warp * d.warp_smem, d.D);
  uint32_t phase = 0;
  const int64_t sb = (int64_t)blockIdx.x * q.n / gridDim.x;
  const int64_t se = (int64_t)(blockIdx.x + 1) * q.n / gridDim.x;
  int64_t s = sb;
  int m = 0;
  const int R = d.R;
  while (s < se) {
    while (q.qoff[m + 1] <= s) ++m;
    const int64_t seg_end = min(se, q.qoff[m + 1]);
    const MapView mv = bind_map(d, m, smem, bar, phase);
    const int64_t nb = (seg_end - s + d.E - 1) / d.E;
    for (int64_t b = warp; b < nb; b += nwarps) {
      const int64_t s0 = s + b * d.E;
      const int E = (int)min((int64_t)d.E, seg_end - s0);
      if (lane < E) {
        double sh_, ch_;
        sincos(q.h[s0 + lane], &sh_, &ch_);
        ws.px[lane] = q.x[s0 + lane];
        ws.py[lane] = q.y[s0 + lane];
        ws.ch[lane] = ch_;
        ws.sh[lane] = sh_;
        ws.list[lane] = lane;
      }
      __syncwarp();
      auto fin = [&](int e, int j, double t, int hit) {
        const int64_t o = (s0 + e) * R + j;
        q.ranges[o] = t;
        if (q.hit_cell) q.hit_cell[o] = hit;
      };
      ray_phase<true>(mv, d, ws, beam, E, fin);
      __syncwarp();
    }
    s = seg_end;
  }
}

}  // namespace sp
