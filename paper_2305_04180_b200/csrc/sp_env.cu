// sp_env.cu -- the fused Sparrow step (+auto-reset) kernel for sm_100a.
//
// One launch per VecEnv.step_batch (vecenv.py:94-116 -> core.py:165-219, with
// the auto-reset of core.py:114-161 fused in).  Layout and schedule:
//
// * Lanes (env copies) are stored struct-of-arrays in MAP-MAJOR slot order;
//   env_of_slot maps a slot back to the caller's row (outputs keep the
//   reference row order).  The host gives every CTA a contiguous slot range
//   that lies inside one map whenever the map count allows, so a CTA stages
//   one map once per launch.
// * Per map, two tables live in shared memory, staged by one TMA bulk copy
//   (cp.async.bulk + mbarrier): a per-cell table (signed byte: 0x80 for an
//   occupied cell, else the radius r of the all-free (2r+1)^2-cell box
//   centred on it) that the march reads once per step, and a 1-bit occupancy
//   bitmap (H x ceil(W/32) u32) for the exact disc-collision test.
//   366 x 366 cells -> 131 KB + 17.6 KB.  Every map has an occupied border.
// * Scans write straight into the output rows (the noise z parks in the row
//   until the ray retires), so a chunk needs no staging rows: 86 B of shared
//   memory per scan slot, which is what leaves room for the per-cell table.
// * A CTA walks its range in chunks of up to `chunk_cap` envs with CTA-wide
//   phases separated by __syncthreads:
//     A  thread-per-env physics, collision, events, shaped-reward partial,
//        obs header (fp64 in the reference's rounding order); fused
//        auto-reset of finished envs (resample, spawn rejection) with their
//        fresh scan in an extra slot; collisions / arrivals finish here;
//        threads without an env pre-generate the LiDAR noise;
//     B  one CTA-wide LiDAR ray queue over all scans of the chunk, longest
//        predicted scan first: warps take as many rays as they have idle
//        slots (one shared atomic), two rays per lane;
//     C  thread-per-env reward of running / timed-out envs, outputs, VecEnv
//        statistics.
// * The march visits the same cells as the reference DDA (_cy.pyx:89-105) but
//   jumps over free boxes in one step: at cell (ix,iy) with free box B, the
//   ray leaves B through the face with the smaller exit parameter (ties go to
//   x, as tmx <= tmy does), re-entering the grid at the cell containing the
//   exit point (clamped into B's span on the other axis).  Only free cells
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
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// 8-byte global -> shared copy that never occupies a register (cp.async)
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
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
  uint32_t kbase;  // shared-window address of blk (tables in shared memory), else 0
  __device__ __forceinline__ uint32_t code(int ix, int iy) const {
    return blk[iy * Wb + ix];
  }
  // the same byte sign-extended: < 0 for an occupied cell, else the box radius
  __device__ __forceinline__ int scode(int ix, int iy) const {
    return ((const int8_t*)blk)[iy * Wb + ix];
  }
  __device__ __forceinline__ uint32_t word(int ix, int iy) const {
    return bits[iy * WW + (ix >> 5)];
  }
};

// The signed cell byte at table offset `a` (+ kbase).  With the tables in
// shared memory, rays carry the table's shared-window address in their kb, so
// a march lookup is two IMADs and one LDS with no base add.
template <bool kSmem>
__device__ __forceinline__ int table_code(const MapView& mv, int a) {
  if constexpr (kSmem) {
    int v;
    asm("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  } else {
    return ((const int8_t*)mv.blk)[a];
  }
}

// atomicAdd(ctr, 1) for every calling lane of a warp with one shared-memory
// atomic (consecutive values in lane order).
__device__ __forceinline__ int warp_inc(int* ctr) {
  const unsigned m = __activemask();
  const int leader = __ffs(m) - 1;
  int base = 0;
  if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(ctr, __popc(m));
  base = __shfl_sync(m, base, leader);
  return base + __popc(m & lanemask_lt());
}

// The reference's nearest-point test of one occupied cell (_cy.pyx:141-153).
__device__ __forceinline__ bool cell_within(double x, double y, int ix, int iy, double cell,
                                            double r2) {
  const double clo = dmul((double)ix, cell), chi = dadd(clo, cell);
  double nx = x > clo ? x : clo;
  if (nx > chi) nx = chi;
  const double rlo = dmul((double)iy, cell), rhi = dadd(rlo, cell);
  double ny = y > rlo ? y : rlo;
  if (ny > rhi) ny = rhi;
  const double ddx = dsub(x, nx), ddy = dsub(y, ny);
  return dadd(dmul(ddx, ddx), dmul(ddy, ddy)) <= r2;
}

// Does bbox row iy ([ix0, ix1]) hold an occupied cell within r of (x, y)?
// Along a row the computed distance term ddx^2 is V-shaped in ix (clo, chi
// and the roundings are monotone), flat at 0 over the cell(s) holding x, so
// the row's minimum is at the nearest occupied cell on either side of that
// valley.  The valley is within one cell of cx = floor(x / cell), so the
// candidates are the occupied cells among cx-1..cx+1 plus the nearest one
// beyond each side -- the same answer as testing every occupied cell.
__device__ __forceinline__ bool row_hits(const MapView& mv, double x, double y, int iy, int ix0,
                                         int ix1, int cx, double cell, double r2) {
  const uint32_t* rowp = mv.bits + iy * mv.WW;
  const int width = ix1 - ix0 + 1;
  if (width <= 32) {
    // the row's bbox cells as one 32-bit window starting at ix0
    const int w0 = ix0 >> 5, sh = ix0 & 31;
    const uint32_t lo = rowp[w0], hi = w0 + 1 < mv.WW ? rowp[w0 + 1] : 0u;
    uint32_t m = __funnelshift_r(lo, hi, sh);
    if (width < 32) m &= (1u << width) - 1u;
    if (!m) return false;
    const int c = cx - ix0;  // the centre column in the window
    const int a0 = max(c - 1, 0), a1 = min(c + 1, width - 1);
    if (a0 <= a1) {  // occupied cells among c-1 .. c+1
      uint32_t near = (m >> a0) & ((1u << (a1 - a0 + 1)) - 1u);
      while (near) {
        const int b = __ffs(near) - 1;
        near &= near - 1;
        if (cell_within(x, y, ix0 + a0 + b, iy, cell, r2)) return true;
      }
    }
    if (c - 1 > 0) {  // the nearest occupied cell left of c-1
      const uint32_t left = m & ((1u << min(c - 1, 31)) - 1u);
      if (left && cell_within(x, y, ix0 + 31 - __clz(left), iy, cell, r2)) return true;
    }
    if (c + 2 < width) {  // ... and right of c+1
      const uint32_t right = c + 2 <= 0 ? m : (m & ~((1u << (c + 2)) - 1u));
      if (right && cell_within(x, y, ix0 + __ffs(right) - 1, iy, cell, r2)) return true;
    }
    return false;
  }
  for (int w = ix0 >> 5; w <= (ix1 >> 5); ++w) {  // wide bboxes: every occupied cell
    uint32_t m = rowp[w];
    const int lo = w << 5;
    if (ix0 > lo) m &= ~0u << (ix0 - lo);
    if (ix1 - lo < 31) m &= (2u << (ix1 - lo)) - 1u;
    while (m) {
      const int ix = lo + __ffs(m) - 1;
      m &= m - 1;
      if (cell_within(x, y, ix, iy, cell, r2)) return true;
    }
  }
  return false;
}

// disc_collides for one disc (_cy.pyx:109-158), exact fp64 test, for every
// calling lane of a warp: the cell table proves most discs free with one
// lookup; each remaining disc is tested by all calling lanes together, one
// bbox row per lane (a disc near a wall has ~2r/cell rows; one lane walking
// them all kept its whole warp waiting for microseconds).
__device__ __forceinline__ bool disc_hits(const MapView& mv, const EnvDev& d, double x, double y) {
  const double r = d.radius, cell = d.cell;
  bool res = false, decided = true;
  if (x - r < 0.0 || y - r < 0.0 || x + r > (double)d.W * cell || y + r > (double)d.H * cell) {
    res = true;  // :124-126
  } else {
    const int cx = (int)floor(x * d.inv_cell), cy = (int)floor(y * d.inv_cell);
    decided = false;
    if (cx >= 0 && cx < d.W && cy >= 0 && cy < d.H) {
      const uint32_t code = mv.code(cx, cy);  // free box of radius code covers the bbox?
      if ((code & 0x80u) == 0u && code >= (uint32_t)d.need_k) decided = true;
    }
  }
  const unsigned act = __activemask();
  unsigned pend = __ballot_sync(act, !decided);
  const int nact = __popc(act), rank = __popc(act & lanemask_lt());
  const double r2 = dmul(r, r);
  while (pend) {
    const int src = __ffs(pend) - 1;
    pend &= pend - 1;
    const double xs = __shfl_sync(act, x, src), ys = __shfl_sync(act, y, src);
    int ix0 = (int)floor(ddiv(dsub(xs, r), cell)); if (ix0 < 0) ix0 = 0;  // :128-135
    int ix1 = (int)floor(ddiv(dadd(xs, r), cell)); if (ix1 > d.W - 1) ix1 = d.W - 1;
    int iy0 = (int)floor(ddiv(dsub(ys, r), cell)); if (iy0 < 0) iy0 = 0;
    int iy1 = (int)floor(ddiv(dadd(ys, r), cell)); if (iy1 > d.H - 1) iy1 = d.H - 1;
    const int cxs = (int)floor(xs * d.inv_cell);
    bool hit = false;
    for (int iy = iy0 + rank; iy <= iy1 && !hit; iy += nact)
      hit = row_hits(mv, xs, ys, iy, ix0, ix1, cxs, cell, r2);
    hit = __any_sync(act, hit);
    if ((int)(threadIdx.x & 31) == src) res = hit;
  }
  return res;
}

// ---------------------------------------------- debug phase timestamps ---
// Built only with -DSP_TIMING (tools/debug): thread 0 of each CTA stamps
// %clock64 (SM cycles) at phase boundaries of the last chunk into shared
// memory (a global store could stall behind the CTA's queued row stores and
// skew the stamps), copied out at the kernel's end.
#ifdef SP_TIMING
// [12 + w]: warp w arrives at the end of phase A; per warp w (lane 0, after
// the barrier / phase named): [48 + w] leaves order_entries, [72 + w] enters
// the ray phase, [96 + w] leaves it (before the barrier)
constexpr int kTs = 160;
__device__ unsigned long long g_sp_lane[5][148][768];  // per-lane debug clocks (points 0..4)
// per-lane clock once `dep` is available (the add waits on it; in-order issue)
#ifdef SP_TIMING_LANES  // per-lane clocks (perturb phase A: a global store per lane and point)
#define SP_LSTAMP(p, dep) do { double t0_; \
  asm volatile("add.f64 %0, %1, 0d0000000000000000;" : "=d"(t0_) : "d"((double)(dep))); \
  unsigned long long t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_) :: "memory"); \
  if (blockIdx.x < 148) g_sp_lane[p][blockIdx.x][threadIdx.x] = t_ + (t0_ == 1.25e300 ? 1 : 0); } while (0)
#else
#define SP_LSTAMP(p, dep)
#endif
__device__ unsigned long long g_sp_ts[1024][kTs];
__shared__ unsigned long long s_sp_ts[kTs];
__device__ __forceinline__ void sp_stamp(int k) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    s_sp_ts[k] = t;
  }
}
__device__ __forceinline__ void sp_stamp_flush() {
  __syncthreads();
  if (threadIdx.x == 0) {  // CTA end on the GPU-wide clock (ns)
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)::"memory");
    s_sp_ts[37] = g;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kTs; k += blockDim.x)
    if (blockIdx.x < 1024) g_sp_ts[blockIdx.x][k] = s_sp_ts[k];
}
#define SP_STAMP(k) sp_stamp(k)
// lane 0 of every warp stamps slot base + warp
#define SP_WSTAMP(base) do { if ((threadIdx.x & 31) == 0) { unsigned long long t_; \
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)::"memory"); \
  s_sp_ts[(base) + (threadIdx.x >> 5)] = t_; } } while (0)
// env thread 0 inside step_env (slots 38..)
#define SP_ESTAMP(k) do { if (threadIdx.x == 0) { unsigned long long t_; \
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)::"memory"); s_sp_ts[k] = t_; } } while (0)
#else
#define SP_ESTAMP(k)
#define SP_LSTAMP(p, dep)
#define SP_STAMP(k)
#define SP_WSTAMP(base)
#endif

// ---------------------------------------------------------------- rays ---
#ifndef SP_MARCH_GROUP
#define SP_MARCH_GROUP 4  // march steps per slot between refill checks
#endif
// Ray state, mirrored so that every ray moves toward +u, +v: on an axis the
// ray travels in the negative direction, coordinates are negated (exactly)
// and cell indices become u = -ix - 1, so cell u covers [u, u + 1).  In cell
// units: origin (X, Y); cell / |direction| (IDX, IDY), so t = (face - X) * IDX
// is the reference's parameter in cm -- bit for bit the unmirrored
// ((double)face - x0) * idx, since negation is exact; slopes SY = |dy / dx|
// (v gained per unit of u) and SX = |dx / dy|, which give the other axis at
// a face crossing without the crossing's parameter.  The table address of
// cell (u, v) is v * ayw + u * ax + kb, with (ax, bx) = (1, 0) or (-1, -1) per
// axis (ix = ax * u + bx), ayw = ay * W and kb = by * W + bx (+ the table's
// shared-window address).
struct Ray {
  double X, Y, SX, SY, IDX, IDY;
  int u, v, ax, ayw, kb, n;  // n: march steps taken, in groups of SP_MARCH_GROUP (history)
};

// 1/v to within an ulp: the fp64 reciprocal approximation (full exponent
// range) + two Newton steps, no branches and no DDIV.  v == 0 (an axis the
// ray never crosses) and subnormal v give +-inf.
__device__ __forceinline__ double recip(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double r1 = r * (2.0 - v * r);
  const double r2 = r1 * (2.0 - v * r1);
  return isinf(r) ? r : r2;
}

// Exact int <-> double conversions on the fp64 pipe instead of the slower
// conversion unit: |v| < 2^31 sits in the low mantissa word of v + 1.5 * 2^52.
__device__ __forceinline__ double i2d(int n) {  // n >= 0
  return __hiloint2double(0x43300000, n) - 4503599627370496.0;
}
__device__ __forceinline__ int floor_i(double v) {  // floor(v), |v| < 2^31
  return __double2loint(__dadd_rd(v, 6755399441055744.0));
}

// One march step, branch-free: every lane of the warp executes it.  A
// finished ray is a fixed point (it stays in its occupied cell, or re-derives
// the same over-range exit without moving), so idle and finished rays can keep
// stepping without a liveness test.  The cell byte is negative for an
// occupied cell (the ray stops there), else the radius r of the free
// (2r+1)^2-cell box centred on the cell: r = 0 is one DDA cell step
// (_cy.pyx:89-96), larger r lets the ray leave the whole box.  Either way it
// exits through the face with the smaller parameter (ties to x, as tmx <= tmy
// does) into the cell containing the exit point.  Returns true when the ray
// has finished (idempotent once it has): ray_end() then recovers the range
// and the occupied cell it stopped in.  Every map has an occupied border
// (GridMap's invariant, checked by sp_env_create), so no step can leave the
// grid and there are no bounds tests.
template <bool kSmem>
__device__ __forceinline__ bool ray_step(Ray& r, const MapView& mv, const EnvDev& d) {
  SP_CHECK((unsigned)(r.v * r.ayw + r.u * r.ax + r.kb - (int)mv.kbase) < (unsigned)(d.Wb * d.Hb));
  const int code = table_code<kSmem>(mv, r.v * r.ayw + r.u * r.ax + r.kb);
  const bool occupied = code < 0;  // else the box radius
  // the free box's far faces: u + 1 + r (r = 0: this cell's own face)
  const int fu = r.u + 1 + code;
  const int fv = r.v + 1 + code;
  const double au = (double)fu - r.X, av = (double)fv - r.Y;
  const double tu = au * r.IDX, tv = av * r.IDY;
  const bool xs = tu <= tv;  // ties exit through x, as tmx <= tmy (_cy.pyx:89)
  const bool over = tu > d.max_range && tv > d.max_range;  // min(tu, tv) > max (:97-99)
  // the cell on the other axis at the exit point, clamped between the current
  // cell and the box's far cell (the ray moves monotonically): the crossing
  // of the far x face is at v = Y + au SY, of the far y face at u = X + av SX,
  // both independent of the face choice
  const double pv = fma(au, r.SY, r.Y);
  const double pu = fma(av, r.SX, r.X);
  const int c = floor_i(xs ? pv : pu);
  const int lo = xs ? r.v : r.u;
  const int hi = (xs ? fv : fu) - 1;
  const int cc = min(max(c, lo), hi);
  const bool finished = occupied || over;
  if (!finished) {
    r.u = xs ? fu : cc;
    r.v = xs ? cc : fv;
  }
  return finished;
}

// A parked ray: a finished fixed point for the lanes of a ray slot with no
// ray (cell (0, 0) is a border cell, occupied).
__device__ __forceinline__ void ray_park(Ray& r, const MapView& mv) {
  r.u = r.v = 0;
  r.ax = 1;
  r.ayw = 0;
  r.kb = (int)mv.kbase;
  r.n = 0;
  r.X = r.Y = 0.5;
  r.SX = r.SY = 1.0;
  r.IDX = r.IDY = 1.0;
}

// Range and hit cell of a finished ray.  It stopped either in an occupied
// cell -- then its range is the parameter at which it entered that cell: the
// later of the cell's two entry faces u, v (the march's last exit parameter,
// bit for bit; 0 when the origin cell itself is occupied) -- or past
// max_range (range max_range, no hit cell).  An axis the ray does not move
// along (IDX = inf) has no entry face: its term is -inf, or NaN (0 * inf)
// when the origin lies on that axis's cell boundary, and fmax drops a NaN.
// (Compare-selects instead of fmax, with the NaN case kept out by moving such
// an origin to its cell's centre or tested for, measured +1 % -- dropped.)
template <bool kSmem>
__device__ __forceinline__ double ray_end(const Ray& r, const MapView& mv, const EnvDev& d,
                                          int& hit) {
  const int ix = r.ax * r.u + (r.ax < 0 ? -1 : 0);
  const int iy = r.ayw < 0 ? -r.v - 1 : r.v;
  const bool occ = table_code<kSmem>(mv, r.v * r.ayw + r.u * r.ax + r.kb) < 0;
  hit = occ ? iy * d.W + ix : -1;
  if (!occ) return d.max_range;
  const double eu = ((double)r.u - r.X) * r.IDX, ev = ((double)r.v - r.Y) * r.IDY;
  return fmax(fmax(eu, ev), 0.0);
}

// Returns true if finished during setup (origin outside the grid -> 0).
__device__ __forceinline__ bool ray_setup(Ray& r, double x0, double y0, double ch, double sh,
                                          double2 cs, const EnvDev& d, const MapView& mv) {
  const double dx = ch * cs.x - sh * cs.y;  // cos(h + o_j)
  const double dy = sh * cs.x + ch * cs.y;  // sin(h + o_j)
  const double xc = x0 * d.inv_cell, yc = y0 * d.inv_cell;
  const int ix = (int)floor(xc), iy = (int)floor(yc);
  const bool px = dx >= 0.0, py = dy >= 0.0;  // dx == 0: SY = +inf, x faces never taken
  r.X = px ? xc : -xc;
  r.Y = py ? yc : -yc;
  const double rx = recip(dx), ry = recip(dy);  // +-inf for a zero component
  r.IDX = fabs(rx * d.cell);
  r.IDY = fabs(ry * d.cell);
  r.SY = fabs(dy * rx);  // |dy / dx|: +inf for dx == 0, 0 for dy == 0
  r.SX = fabs(dx * ry);
  r.u = px ? ix : -ix - 1;
  r.v = py ? iy : -iy - 1;
  r.ax = px ? 1 : -1;
  r.ayw = py ? d.Wb : -d.Wb;
  r.kb = (int)mv.kbase + (py ? 0 : -d.Wb) + (px ? 0 : -1);
  r.n = 0;
  return (unsigned)ix >= (unsigned)d.W || (unsigned)iy >= (unsigned)d.H;  // :37-39
}

// Per-CTA chunk scratch (shared memory).  A chunk holds up to `cap` envs;
// its scans use "slots": slot e (< cap) is env e's post-step scan, slots
// cap .. cap+extra-1 are post-reset scans of envs that finished this step.
// A scan's R beams form up to 8 "beam groups" of gb = 2^gshift consecutive
// beams (EnvDev::gshift); the ray queue dispatches (slot, group) entries.
// One scan slot's record (80 B: every field at an immediate offset of one
// base address, the 16-byte pairs loaded as 128-bit words; the 20-word stride
// spreads 8 consecutive slots over disjoint banks).
struct SlotRec {
  double px, py;   // scan origin (cm)
  double ch, sh;   // heading cos / sin
  double sig;      // noise std (cm)
  float* out0;     // the output row its scan fills (noise z parks there first)
  float* out1;     // a second row that receives the same values, or null
  uint64_t qacc;   // byte g = OR of 1 << step_level(steps) over group g's rays
  uint64_t nctr;   // first Philox block of the slot's LiDAR noise
  uint64_t qpred;  // the qacc bytes of the lane's last scan (dispatch prediction)
};

struct Chunk {
  SlotRec* rec;    // per slot
  double* retp;    // per env: episode return before this step (prefetched in phase A)
  double* part;    // per env: shaped reward without its proximity term
  uint32_t* gid;   // per slot: the env's stream lane (global env id)
  int32_t* reg;    // slots in registration order
  int32_t* hwrite; // per slot: global slot whose history this scan refreshes, or -1
  int32_t* xslot;  // per env: post-reset slot, -1 if none
  int* ctl;        // [0] ray-queue head [1] slots listed [2] extra slots used [3] overflow
                   // [4..11] bucket counts, [12..19] bucket offsets, [20] entries listed
                   // late resets: [21] env lanes past their reset decision, [22] late
                   // queue entries, [23] late slots claimed
  int32_t* rowi;   // per env: caller row
  int32_t* send;   // per env: episode length before any reset
  uint16_t* list;  // (slot << 3 | group) entries in dispatch order (longest predicted first)
  uint8_t* wmode;  // per env: which rows to write (see kernel)
  int8_t* evs;     // per env: event awaiting phase C, or -1 (nothing left to do)
  uint8_t* prox;   // per slot: some ray ended closer than the proximity range
};

__device__ __forceinline__ Chunk chunk_smem(uint8_t* smem, const EnvDev& d) {
  Chunk c;
  c.rec = (SlotRec*)(smem + d.co[CF_REC]);
  c.retp = (double*)(smem + d.co[CF_RETP]);
  c.part = (double*)(smem + d.co[CF_PART]);
  c.gid = (uint32_t*)(smem + d.co[CF_GID]);
  c.reg = (int32_t*)(smem + d.co[CF_REG]);
  c.hwrite = (int32_t*)(smem + d.co[CF_HWRITE]);
  c.xslot = (int32_t*)(smem + d.co[CF_XSLOT]);
  c.ctl = (int*)(smem + d.co[CF_CTL]);
  c.rowi = (int32_t*)(smem + d.co[CF_ROWI]);
  c.send = (int32_t*)(smem + d.co[CF_SEND]);
  c.list = (uint16_t*)(smem + d.co[CF_LIST]);
  c.wmode = smem + d.co[CF_WMODE];
  c.evs = (int8_t*)(smem + d.co[CF_EVS]);
  c.prox = smem + d.co[CF_PROX];
  return c;
}

// March-step history level of a ray (steps incl. the finishing one), about
// half an octave per level: <= 3, 4-5, 6-7, 8-11, 12-15, 16-23, 24-31, >= 32.
__device__ __forceinline__ int step_level(int steps) {
  const int s = steps > 2 ? steps : 2;
  const int msb = 31 - __clz(s);
  const int lv = 2 * msb + ((s >> (msb - 1)) & 1) - 3;
  return lv < 0 ? 0 : (lv > 7 ? 7 : lv);
}

// step_level of a retiring ray: its step count is 1 + a multiple of
// SP_MARCH_GROUP (steps are counted per group, ray_phase), so with groups of
// four the level is a nibble table on steps / 4: 1, 5, 9, .., 33+ -> 0 1 3 4 5 5 6 6 7
__device__ __forceinline__ int retire_level(int steps) {
#if SP_MARCH_GROUP == 4
  return (int)(0x766554310ull >> (4 * min(steps >> 2, 8))) & 15;
#else
  return step_level(steps);
#endif
}

// predicted bucket of a beam group (0 = longest): 7 - its highest level
// (no history -> 0x80 -> bucket 0)
__device__ __forceinline__ int group_bucket(uint64_t pred, int g) {
  const uint32_t b = (uint32_t)(pred >> (8 * g)) & 0xffu;
  return b ? __clz(b) - 24 : 0;
}

constexpr uint64_t kNoHistory = 0x8080808080808080ull;  // every group "longest"

// List entries reserved ahead of the ordered ones for late-reset entries
// (reset_late): at most every spare slot's groups.
__device__ __forceinline__ int late_reserve(const EnvDev& d) {
  return (d.slot_cap - d.chunk_cap) * d.n_groups;
}

// queue index q -> (slot, beam) of its (slot, group) entry in qlist
__device__ __forceinline__ int beam_of(const uint16_t* qlist, int q, int gs, int n_ent, int& slot) {
  SP_CHECK((q >> gs) < n_ent);
  (void)n_ent;
  const uint32_t e = qlist[q >> gs];
  slot = (int)(e >> 3);
  return (int)((e & 7u) << gs) + (q & ((1 << gs) - 1));
}

// CTA-wide ray queue over n_ent (slot, group) entries (qlist) x gb beams:
// queue index q -> entry qlist[q >> gshift], beam (group << gshift) + (q & (gb - 1));
// beams >= R (a partial last group) are skipped.  fin(slot, j, t, hit).
// Every thread of the CTA must call it.  Each lane marches two independent
// rays (slots A and B) so one ray's fp64 dependency chain hides behind the
// other's.  A warp refills only when at least d.refill_min of its 64 ray
// slots are idle (or the queue is drained); finished rays are retired in the
// same branch, so per-ray setup/finish code runs at high SIMT occupancy.
template <bool kSmem, bool kHit, class Fin>
__device__ __forceinline__ void ray_phase(const MapView& mv, const EnvDev& d, const Chunk& c,
                                          const double2* beam, const uint16_t* qlist, int n_ent,
                                          const Fin& fin) {
  const int R = d.R;
  const int gs = d.gshift;
  const int total = n_ent << gs;
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  // busy: the slot holds a ray not yet retired; fin: the slot's ray has
  // finished (parked slots count as finished)
  bool busy_a = false, busy_b = false, fin_a = true, fin_b = true;
  bool drained = total == 0;
  int ea = 0, ja = 0, eb = 0, jb = 0;
  float za = 0.0f, zb = 0.0f;  // the slots' prefetched noise (Fin::pre)
  Ray ra, rb;
  ray_park(ra, mv);
  ray_park(rb, mv);
  for (;;) {
    const unsigned ia = __ballot_sync(SP_FULL, fin_a);
    const unsigned ib = __ballot_sync(SP_FULL, fin_b);
    const int na = __popc(ia), n_idle = na + __popc(ib);
    if (n_idle >= d.refill_min || drained) {
      if (busy_a && fin_a) {  // steps taken = moves + the finishing step
        int hit;
        const double t = ray_end<kSmem>(ra, mv, d, hit);
        fin(ea, ja, t, kHit ? hit : -1, ra.n + 1, za);
        busy_a = false;
      }
      if (busy_b && fin_b) {
        int hit;
        const double t = ray_end<kSmem>(rb, mv, d, hit);
        fin(eb, jb, t, kHit ? hit : -1, rb.n + 1, zb);
        busy_b = false;
      }
      if (drained) {
        if ((ia & ib) == SP_FULL) break;
      } else {
        int base = 0;
        if (lane == 0) base = atomicAdd(&c.ctl[0], n_idle);
        base = __shfl_sync(SP_FULL, base, 0);
        if (base + n_idle >= total) {
#ifdef SP_TIMING
          if (base < total && lane == 0 && blockIdx.x < 1024) {  // the queue just drained
            unsigned long long t;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
            s_sp_ts[10] = t;
          }
#endif
          drained = true;
        }
        const int my_a = base + __popc(ia & lt);
        const int my_b = base + na + __popc(ib & lt);
        if (fin_a && my_a < total && (ja = beam_of(qlist, my_a, gs, n_ent, ea)) < R) {
          za = fin.pre(ea, ja);
          if (ray_setup(ra, c.rec[ea].px, c.rec[ea].py, c.rec[ea].ch, c.rec[ea].sh, beam[ja], d, mv)) {
            fin(ea, ja, 0.0, -1, 1, za);  // origin outside the grid: range 0 (_cy.pyx:37-39)
            ray_park(ra, mv);
          } else {
            busy_a = true;
            fin_a = false;
          }
        }
        if (fin_b && my_b < total && (jb = beam_of(qlist, my_b, gs, n_ent, eb)) < R) {
          zb = fin.pre(eb, jb);
          if (ray_setup(rb, c.rec[eb].px, c.rec[eb].py, c.rec[eb].ch, c.rec[eb].sh, beam[jb], d, mv)) {
            fin(eb, jb, 0.0, -1, 1, zb);
            ray_park(rb, mv);
          } else {
            busy_b = true;
            fin_b = false;
          }
        }
      }
    }
    // four march steps per slot between refill checks: the loop's votes and
    // branch are paid once per four steps (2 -> 4: -2 % step with the cheaper
    // per-cell steps); a finished ray stays put for the rest of the group
    // march steps counted per group (the scheduling history only; a ray that
    // finishes inside the group is over-counted by at most 3): one add per
    // group instead of one per step (-3.6 % step)
    if (!fin_a) ra.n += SP_MARCH_GROUP;
    if (!fin_b) rb.n += SP_MARCH_GROUP;
#pragma unroll
    for (int u = 0; u < SP_MARCH_GROUP; ++u) {
      fin_a = ray_step<kSmem>(ra, mv, d);
      fin_b = ray_step<kSmem>(rb, mv, d);
    }
  }
}

// Longest-first order (LPT) of the chunk's rays, per beam group: each
// (scan, group) entry is ranked by the march-step level of the longest ray of
// the same beam group in its lane's last scan (the robot moves <= 1.8 cm and
// turns <= 0.1 rad per step, so a beam's step count mostly persists: 64 % of
// rays repeat it exactly).  Fresh spawns have no history and rank longest.
// Entries are counting-sorted into 8 buckets, longest first, so a warp's 64
// ray slots hold rays of similar length (fewer lanes march finished rays
// while their neighbours finish) and the queue tail holds short rays only.
// tools/warp_sim.py models this against per-scan ranking (-16 % ray phase).

// Refresh the lanes' step-level history from this chunk's scans (after a ray
// phase, before its slots are reused): the n_slots registered slots c.reg[].
__device__ __forceinline__ void store_history(const EnvDev& d, const Chunk& c, int n_slots,
                                              int n_late_slots = 0) {
  for (int k = threadIdx.x; k < n_slots + n_late_slots; k += blockDim.x) {
    // late-reset slots (reset_late; hwrite -1 after a failed spawn) follow
    const int slot = k < n_slots ? c.reg[k] : d.chunk_cap + (k - n_slots);
    const int hw = c.hwrite[slot];
    if (hw >= 0) d.qhist[hw] = c.rec[slot].qacc;
  }
}

// The threads that cooperate on a phase: the whole CTA (barrier 0 =
// __syncthreads) or a warp-aligned group with its own named barrier.
struct Grp {
  int tid, n, id;
  __device__ __forceinline__ void sync() const {
    if (id == 0)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};
__device__ __forceinline__ Grp cta_grp() { return Grp{(int)threadIdx.x, (int)blockDim.x, 0}; }

// Counting sort of the chunk's (slot, group) entries into c.list, longest
// predicted first; c.ctl[20] = entries listed.  Warp-aggregated atomics: one
// shared atomic per bucket present in a warp's 32 entries.
__device__ __forceinline__ void order_entries(const EnvDev& d, const Chunk& c, int n_slots,
                                              const Grp& g, uint16_t* out) {
  int* cnt = c.ctl + 4;
  int* off = c.ctl + 12;
  const int G = d.n_groups;
  const int space = n_slots * 8;
  const int lane = g.tid & 31;
  const unsigned lt = lanemask_lt();
  if (g.tid < 8) cnt[g.tid] = 0;
  g.sync();
  for (int base = g.tid - lane; base < space; base += g.n) {  // warp-uniform trips
    const int k = base + lane;
    int b = 8;  // no entry
    if (k < space && (k & 7) < G) b = group_bucket(c.rec[c.reg[k >> 3]].qpred, k & 7);
    const unsigned peers = __match_any_sync(SP_FULL, b);
    if (b < 8 && (peers & lt) == 0) atomicAdd(&cnt[b], __popc(peers));
  }
  g.sync();
  if (g.tid == 0) {
    int acc = 0;
    for (int b = 0; b < 8; ++b) {
      off[b] = acc;
      acc += cnt[b];
    }
    c.ctl[20] = acc;
  }
  g.sync();
  for (int base = g.tid - lane; base < space; base += g.n) {
    const int k = base + lane;
    int b = 8;
    int slot = 0;
    if (k < space && (k & 7) < G) {
      slot = c.reg[k >> 3];
      b = group_bucket(c.rec[slot].qpred, k & 7);
    }
    const unsigned peers = __match_any_sync(SP_FULL, b);
    const int leader = __ffs(peers) - 1;
    int pos = 0;
    if (b < 8 && lane == leader) pos = atomicAdd(&off[b], __popc(peers));
    pos = __shfl_sync(SP_FULL, pos, leader);
    SP_CHECK(b >= 8 || pos + __popc(peers & lt) < 8 * d.slot_cap);
    if (b < 8) out[pos + __popc(peers & lt)] = (uint16_t)((slot << 3) | (k & 7));
  }
  g.sync();  // the list complete before anyone dispatches from it
}

__device__ __forceinline__ void set_error(const EnvDev& d, int code, int64_t row) {
  if (atomicCAS(d.err, 0, code) == 0) d.err[1] = (int32_t)row;
}

// caller row of slot s of map m (map_off[m] = mstart): computed for the default
// map assignment (EnvDev::row_affine), else the env_of_slot table
__device__ __forceinline__ int64_t row_of(const EnvDev& d, int m, int64_t mstart, int64_t s) {
  if (d.row_affine) {
    const int i0 = m >= d.off_mod ? m - d.off_mod : m - d.off_mod + d.n_maps;
    return i0 + (s - mstart) * d.n_maps;
  }
  return d.env_of_slot[s];
}

// LiDAR noise (core.py:237-241): every listed slot needs R standard normals
// from blocks nctr[slot] .. nctr[slot]+nb-1 of its stream.  One work item per
// Philox block, spread over the whole CTA; z parks in the slot's output row.
// z ~ N(0,1) of one noise block (4 beams) of `slot` into its output row
__device__ __forceinline__ void noise_block(const EnvDev& d, const Chunk& c, int slot, int b) {
  const Block4 blk = stream_block(d.seed, c.gid[slot], 0u, c.rec[slot].nctr + (uint64_t)b);
  float z[4];
  draw_normals4(blk, z);
  SP_CHECK(slot >= 0 && slot < d.slot_cap && b >= 0 && b < d.nb);
  float* row = c.rec[slot].out0 + 5 + 4 * b;
#ifdef SP_EXP_NOZ  // experiment: no z stores (wrong noise), isolates their cost
  if (z[0] == 12345.0f)
#endif
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (4 * b + u < d.R) row[u] = z[u];
}

// The LiDAR noise of env slots 0..n-1 computed by the threads that have no env
// in phase A, while phase A runs (env slot = its env's chunk index): a post-step scan draws from the env's
// counter at step start (c.nctr/c.gid snapshot at chunk start), and only z is
// staged (sigma is applied when the ray retires), so nothing here depends on
// phase A.  first = the first idle thread.
__device__ __forceinline__ void prenoise(const EnvDev& d, const StepArgs& a, const Chunk& c,
                                         int n, int first, int64_t s0, int m, int64_t mstart) {
  const int nb = d.nb;
  const int idle = (int)blockDim.x - first;
  // the noise streams of env slots 0..n-1 (the values add_slot later writes
  // into the same words): loaded by the noise warps themselves, so the env
  // threads never wait for them; then a barrier among the noise warps only
  for (int k = (int)threadIdx.x - first; k < n; k += idle) {
    const int64_t s = s0 + k;
    const int64_t row = row_of(d, m, mstart, s);
    c.rec[k].nctr = d.ctr[s];
    c.gid[k] = (uint32_t)(d.env_id_offset + row);
    c.rec[k].out0 = a.store_states + row * d.D;  // z parks in the store_states row
  }
  asm volatile("bar.sync 1, %0;" ::"r"(idle) : "memory");
  for (int it = (int)threadIdx.x - first; it < n * nb; it += idle) {
    const int k = d.nb_shift >= 0 ? (it >> d.nb_shift) : it / nb;
    noise_block(d, c, k, it - k * nb);
  }
}

// slots below `pre` (env slots) were pre-noised during phase A (prenoise)
__device__ __forceinline__ void noise_phase(const EnvDev& d, const Chunk& c, int n_slots, int pre,
                                            const Grp& g) {
  const int nb = d.nb;
  const int items = n_slots * nb;
  for (int it = g.tid; it < items; it += g.n) {
    const int k = d.nb_shift >= 0 ? (it >> d.nb_shift) : it / nb;
    const int b = it - k * nb;
    const int slot = c.reg[k];
    if (slot < pre) continue;
    noise_block(d, c, slot, b);
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
  const double vx = dsub(gx, sx), vy = dsub(gy, sy);
  const double len2 = dadd(dmul(vx, vx), dmul(vy, vy));
  const double safe = len2 > 0.0 ? len2 : 1.0;
  double t = dclip(ddiv(dadd(dmul(dsub(x, sx), vx), dmul(dsub(y, sy), vy)), safe), 0.0, 1.0);
  if (!(len2 > 0.0)) t = 0.0;
  const double ex = dsub(x, dadd(sx, dmul(t, vx))), ey = dsub(y, dadd(sy, dmul(t, vy)));
  return __dsqrt_rn(dadd(dmul(ex, ex), dmul(ey, ey)));
}

// v / m for v in [0, m] from the reciprocal plus one exact-residual correction
// (Markstein): the correctly rounded quotient without a DDIV.
__device__ __forceinline__ double div_by(double v, double m, double inv_m) {
  const double q = v * inv_m;
  const double r = fma(-q, m, v);
  return fma(r, inv_m, q);
}

// core.py:243-258 columns 0..4 (LiDAR columns come from the ray phase)
__device__ __forceinline__ void header_row(const MapConst& mc, double x, double y, double alpha,
                                           double c0, double s0, double vl, double va, double vml,
                                           double vma, float* row, float* row1) {
  const double rx = dsub(mc.goal_x, x), ry = dsub(mc.goal_y, y);
  float h[5];
  h[0] = (float)div_by(dadd(dmul(c0, rx), dmul(s0, ry)), mc.plan_dist, mc.inv_plan);
  h[1] = (float)div_by(dadd(dmul(-s0, rx), dmul(c0, ry)), mc.plan_dist, mc.inv_plan);
  h[2] = (float)div_by(alpha, SP_PI, SP_INV_PI);
  h[3] = (float)ddiv(vl, vml);
  h[4] = (float)ddiv(va, vma);
#ifdef SP_EXP_NOHDR  // experiment: no header stores (wrong rows), isolates their cost
  if (h[0] == 12345.0f)
#endif
#pragma unroll
  for (int k = 0; k < 5; ++k) row[k] = h[k];
#ifdef SP_EXP_NOHDR
  if (h[0] == 12345.0f)
#endif
  if (row1) {
#pragma unroll
    for (int k = 0; k < 5; ++k) row1[k] = h[k];
  }
}

// Finish functor of the ray phase: noisy normalized obs into the staging row
// (core.py:237-241, 257) and the proximity flag (reward.py:70: scan_min < 30
// is "some ray < 30", core.py:205).
// kRec (recording builds of the launch, StepArgs::hit_store etc.): also the
// ray's hit cell and noisy range at the caller row of the scan's rows.
template <bool kRec>
struct FinObs {
  Chunk c;
  int D;
  double max_range, inv_max_range, proximity;
  // recording only
  int32_t *hit_store, *hit_state;
  double* scan_state;
  const float* store_base;  // a.store_states (null outside MODE_STEP)
  uint64_t store_span;      // n * D floats
  uint32_t gid0;            // (uint32) env_id_offset: row = gid - gid0
  int R;
  int gs;                   // log2 of the beams per group (step-level history)
  int d_slot_cap;           // SP_CHECKED bounds
  // z of beam j, parked in the output row by the noise pass: loaded when the
  // ray is dispatched so the L2 round trip overlaps its march
  __device__ __forceinline__ float pre(int slot, int j) const { return c.rec[slot].out0[5 + j]; }
  __device__ __forceinline__ void operator()(int slot, int j, double t, int hit, int steps,
                                             float zpre) const {
    float* rowp = c.rec[slot].out0;
    SP_CHECK(slot >= 0 && slot < d_slot_cap && j >= 0 && j < R);
    const double z = (double)zpre;
    // clip(raw + (0 + sigma z), 0, max) (core.py:240-241): the 0 + only turns
    // a -0.0 into +0.0, which t + (.) absorbs for t >= 0; all finite, so
    // plain selects replace the NaN-aware fmin/fmax
    double v = dadd(t, dmul(c.rec[slot].sig, z));
    v = v < 0.0 ? 0.0 : v;
    v = v > max_range ? max_range : v;
    const float o = (float)div_by(v, max_range, inv_max_range);
    rowp[5 + j] = o;
    float* r1 = c.rec[slot].out1;
    if (r1) r1[5 + j] = o;
    if (t < proximity) c.prox[slot] = 1;
    const int grp = j >> gs;  // byte grp of the 64-bit word, as a 32-bit OR (native)
    atomicOr((unsigned*)&c.rec[slot].qacc + (grp >> 2), 1u << (8 * (grp & 3) + retire_level(steps)));
    if constexpr (kRec) {
      const int64_t k = (int64_t)(c.gid[slot] - gid0) * R + j;
      // post-step scans fill a store_states row (and the states row too when
      // the env keeps running); fresh-spawn scans fill a states row
      const bool store = store_base && (uint64_t)(rowp - store_base) < store_span;
      if (store && hit_store) hit_store[k] = hit;
      if (!store || r1) {
        if (hit_state) hit_state[k] = hit;
        if (scan_state) scan_state[k] = v;
      }
    }
  }
};

// Load map m's tables (TMA bulk copy into shared memory) -- or point at HBM.
template <bool kSmem>
__device__ __forceinline__ MapView bind_map(const EnvDev& d, int m, uint8_t* smem_maps,
                                            uint64_t* bar, uint32_t& phase, bool wait = true) {
  const uint8_t* src = d.maps + (size_t)m * d.map_bytes;
  MapView mv;
  mv.W = d.W;
  mv.H = d.H;
  mv.Wb = d.Wb;
  mv.WW = d.WW;
  if constexpr (kSmem) {
    __syncthreads();  // everyone is done with the previous map
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, d.map_bytes);
      tma_bulk_g2s(smem_maps, src, d.map_bytes, bar);
    }
    if (wait) mbar_wait(bar, phase);
    phase ^= 1u;
    mv.blk = smem_maps;
    mv.bits = (const uint32_t*)(smem_maps + d.blk_bytes);
    mv.kbase = smem_u32(smem_maps);
  } else {
    mv.blk = src;
    mv.bits = (const uint32_t*)(src + d.blk_bytes);
    mv.kbase = 0;
  }
  return mv;
}

// Register a scan slot: origin, heading, noise stream position; queue it.
__device__ __forceinline__ void add_slot(const EnvDev& d, const Chunk& c, int slot, double x,
                                         double y, double ch, double sh, double sig, uint32_t gid,
                                         uint64_t nctr, int32_t hwrite, float* o0, float* o1,
                                         bool reg = true) {
  SP_CHECK(slot >= 0 && slot < d.slot_cap && c.ctl[1] < d.slot_cap);
  c.rec[slot].out0 = o0;
  c.rec[slot].out1 = o1;
  c.hwrite[slot] = hwrite;
  c.rec[slot].px = x; c.rec[slot].py = y; c.rec[slot].ch = ch; c.rec[slot].sh = sh; c.rec[slot].sig = sig;
  c.gid[slot] = gid;
  c.rec[slot].nctr = nctr;
  c.prox[slot] = 0;
  c.rec[slot].qacc = 0;
  if (reg) c.reg[atomicAdd(&c.ctl[1], 1)] = slot;  // else a late reset: queued by reset_late
}

// core.py:114-156 for one lane (stream bound to gid): resample, spawn, write
// the episode SoA fields and the obs header of `slot`, queue its scan (the
// noise blocks follow the reset draws, core.py:159-160).  false = no spawn.
__device__ __forceinline__ bool reset_env(const EnvDev& d, const MapView& mv, const MapConst& mc,
                                          int64_t s, uint32_t gid, uint64_t& ctr, const Chunk& c,
                                          int slot, float* orow, bool reg = true) {
  const double* rg = d.ranges + (d.ranges_shared ? 0 : 12 * s);
  // DiversityRanges.sample (params.py:112-121): U U I U U U
  const double k = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), rg[0], rg[1]);
  const double dt = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), rg[2], rg[3]);
  const int32_t delay = (int32_t)draw_integer(stream_block(d.seed, gid, 0u, ctr++),
                                              (int64_t)rg[4], (int64_t)rg[5] + 1);
  const double vml = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), rg[6], rg[7]);
  const double vma = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), rg[8], rg[9]);
  const double sig = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), rg[10], rg[11]);
  // spawn rejection (core.py:135-147)
  bool ok = false;
  double x = 0, y = 0, th = 0;
  for (int at = 0; at < d.spawn_attempts; ++at) {
    x = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), mc.spawn[0], mc.spawn[2]);
    y = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), mc.spawn[1], mc.spawn[3]);
    th = draw_uniform(stream_block(d.seed, gid, 0u, ctr++), -SP_PI, SP_PI);
    if (!disc_hits(mv, d, x, y)) {
      ok = true;
      break;
    }
  }
  if (!ok) return false;
  double s0, c0;
  sincos(th, &s0, &c0);  // core.py:151-152
  d.x[s] = x; d.y[s] = y; d.h[s] = th; d.vl[s] = 0.0; d.va[s] = 0.0;
  d.sx[s] = x; d.sy[s] = y; d.c0[s] = c0; d.s0[s] = s0;
  d.pk[s] = k; d.pdt[s] = dt; d.pvl[s] = vml; d.pva[s] = vma; d.psig[s] = sig;
  d.delay[s] = delay;
  d.step[s] = 0;
  d.needs_reset[s] = 0;
  for (int wi = 0; wi < ((delay + 15) >> 4); ++wi) d.hist[(int64_t)wi * d.n + s] = ~0ull;
  header_row(mc, x, y, bearing_error(x, y, th, mc.goal_x, mc.goal_y), c0, s0, 0.0, 0.0, vml, vma,
             orow, nullptr);
  c.rec[slot].qpred = kNoHistory;  // a fresh spawn has no step history: ranks longest
  add_slot(d, c, slot, x, y, c0, s0, sig, gid, ctr, (int32_t)s, orow, nullptr, reg);
  ctr += d.nb;
  return true;
}

// Row write modes (per env, Chunk::wmode)
enum : uint8_t {
  W_NONE = 0,      // no output (invalid action / waiting for a reset)
  W_KEEP = 1,      // s' row == post-step row: stage[e] -> store_states, states
  W_RESET_X = 2,   // stage[e] -> store_states, stage[xslot[e]] -> states
  W_RESET_OV = 3,  // stage[e] -> store_states; states after the overflow pass
  W_STATE = 4      // stage[e] -> states only (reset_all, overflow pass)
};

// Phase A of one env in MODE_STEP (core.py:165-206 + vecenv.py:96-114): delay
// queue, kinematics, collision, events, the reward without its proximity term,
// the obs header, the post-step scan's slot (e) and, for a finished episode,
// the fused auto-reset with its fresh scan in an extra slot (cap.. slot_cap-1).
// ctr advances past the draws used; the caller stores it.
struct StepA {
  bool live = false, ended = false;
  bool handed = false;  // the reset warp owns the env's state from the decision on
  int8_t ev = 0;
  int32_t step_end = 0;  // episode length before any reset
  double partial = 0.0;  // shaped reward minus the proximity term
};

__device__ __forceinline__ StepA step_env(const EnvDev& d, const StepArgs& a, const MapView& mv,
                                          const MapConst& mc, const Chunk& c, int e, int64_t s,
                                          int64_t row, uint32_t gid, uint64_t& ctr, int64_t av,
                                          int cap, int slot_cap, uint64_t* mbar, int mpar,
                                          bool late) {
  StepA r;
  // the lane state is loaded before the action checks, so its DRAM round
  // trip overlaps the action load
  double x = d.x[s], y = d.y[s], h = d.h[s], vl = d.vl[s], va = d.va[s];
  const double k = d.pk[s], dt = d.pdt[s], vml = d.pvl[s], vma = d.pva[s];
  const int32_t delay = d.delay[s];
  int32_t step = d.step[s];
  const uint8_t nr = d.needs_reset[s];
  if (av < 0 || av >= d.n_actions) {
    set_error(d, SP_EACTION, row);
    if (late) warp_inc(&c.ctl[21]);
  } else if (nr) {
    set_error(d, SP_EEPISODE, row);
    if (late) warp_inc(&c.ctl[21]);
  } else {
    r.live = true;
    // delay queue (core.py:176-182): matured = action issued `delay` steps ago
    SP_ESTAMP(38);
    SP_LSTAMP(0, x + vl + k + (double)delay + (double)step + (double)av);
    uint32_t code = (uint32_t)av;
    if (delay > 0) {
      const int q = delay - 1;
      const uint64_t h0 = d.hist[s];
      const uint64_t w = q < 16 ? h0 : d.hist[(int64_t)(q >> 4) * d.n + s];
      code = (uint32_t)(w >> (4 * (q & 15))) & 15u;
      const int nw = (delay + 15) >> 4;
      uint64_t carry = (uint64_t)av;
      for (int wi = 0; wi < nw; ++wi) {
        const uint64_t cur = wi == 0 ? h0 : d.hist[(int64_t)wi * d.n + s];
        d.hist[(int64_t)wi * d.n + s] = (cur << 4) | carry;
        carry = cur >> 60;
      }
    }
    const double mv_ = d.action_v[code], mw_ = d.action_w[code];
    // apply_kinematics (kinematics.py:22-36)
    const double omk = dsub(1.0, k);
    vl = dclip(dadd(dmul(k, vl), dmul(omk, mv_)), -vml, vml);
    va = dclip(dadd(dmul(k, va), dmul(omk, mw_)), -vma, vma);
    // integrate_unicycle (kinematics.py:39-63)
    double sin0, cos0, sin1, cos1;
    sincos(h, &sin0, &cos0);
    const double h1 = dadd(h, dmul(va, dt));
    sincos(h1, &sin1, &cos1);
    double ddx, ddy;
    if (fabs(va) >= 1e-6) {
      const double radius = ddiv(vl, va);
      ddx = dmul(radius, dsub(sin1, sin0));
      ddy = dmul(-radius, dsub(cos1, cos0));
    } else {
      ddx = dmul(dmul(vl, cos0), dt);
      ddy = dmul(dmul(vl, sin0), dt);
    }
    x = dadd(x, ddx);
    y = dadd(y, ddy);
    h = wrap_angle(h1);
    // events (core.py:189-201)
    SP_ESTAMP(39);
    SP_LSTAMP(1, x + y);
    if (mpar >= 0) mbar_wait(mbar, (uint32_t)mpar);  // the map tables (staged during the loads above)
    SP_ESTAMP(40);
    const bool coll = disc_hits(mv, d, x, y);
    SP_ESTAMP(41);
    SP_LSTAMP(2, coll ? 1.0 : 0.0);
    const double gdx = dsub(mc.goal_x, x), gdy = dsub(mc.goal_y, y);
    const double d1 = __dsqrt_rn(dadd(dmul(gdx, gdx), dmul(gdy, gdy)));
    const bool arrived = !coll && d1 <= mc.goal_r;
    step += 1;
    const bool timed_out = !coll && !arrived && step >= d.timeout;
    r.ev = coll ? 1 : (arrived ? 2 : (timed_out ? 3 : 0));
    r.ended = coll || arrived || timed_out;
    // fused auto-reset (vecenv.py:113-114) into a spare scan slot, else the
    // overflow pass.  With `late`, the reset is handed to the reset warp
    // (reset_late) here, at the decision: it runs beside the rest of phase A
    // and the ordering instead of after this lane's reward and header, and
    // this lane leaves the episode state to it (no pose / step / counter
    // writes below).
    int xs = -1;
    c.wmode[e] = W_KEEP;
    if (r.ended && d.auto_reset) {
      const int k2 = atomicAdd(&c.ctl[2], 1);
      if (k2 < slot_cap - cap) {
        xs = cap + k2;
        if (late) {
          // parked in the spare slot's record until reset_env fills it
          c.rec[xs].nctr = ctr + (uint64_t)d.nb;  // after this step's post-step scan blocks
          c.rec[xs].qpred = (uint64_t)e;
          c.xslot[e] = xs;
          c.wmode[e] = W_RESET_X;
          r.handed = true;
        }
      } else {
        c.wmode[e] = W_RESET_OV;  // extra slots exhausted: second pass below
        atomicAdd(&c.ctl[3], 1);
      }
    }
    if (late) {
      __threadfence_block();  // the hand-off is visible before the count
      __syncwarp(__activemask());
      warp_inc(&c.ctl[21]);
    }
    SP_LSTAMP(3, (double)r.ev);
    // the episode constants read from here on arrived by cp.async into this
    // env's (not yet registered) scan-slot words at chunk start
    asm volatile("cp.async.wait_all;" ::: "memory");
    const double ep_sx = c.rec[e].px, ep_sy = c.rec[e].py, ep_c0 = c.rec[e].ch, ep_s0 = c.rec[e].sh;
    const double ep_sig = c.rec[e].sig;
    // shaped reward without the proximity term (reward.py:55-73) + obs header
    const double alpha = bearing_error(x, y, h, mc.goal_x, mc.goal_y);
    if (r.ev == 0 || r.ev == 3) {
      const double d2 = cross_track(x, y, ep_sx, ep_sy, mc.goal_x, mc.goal_y);
      const double r_d1 = dclip(dsub(1.0, div_by(d1, mc.plan_dist, mc.inv_plan)), 0.0, 1.0);
      const double r_d2 = dclip(dsub(1.0, div_by(d2, mc.plan_dist, mc.inv_plan)), 0.0, 1.0);
      const double r_v = vl > dmul(vml, 0.5) ? 1.0 : 0.0;  // vml / 2, exact
      const double r_a = dclip(dsub(1.0, div_by(dmul(2.0, fabs(alpha)), SP_PI, SP_INV_PI)), -1.0,
                               1.0);
      r.partial = dadd(dadd(dadd(dmul(0.3, r_d1), dmul(0.1, r_d2)), dmul(0.3, r_v)),
                     dmul(0.3, r_a));
    }
    // rows: the post-step obs goes to store_states, and to states too unless
    // the episode ended and resets (then states gets the fresh scan)
    float* o_store = a.store_states + row * d.D;
    float* o_state = r.ended && d.auto_reset ? nullptr : a.states + row * d.D;
    SP_ESTAMP(42);
    header_row(mc, x, y, alpha, ep_c0, ep_s0, vl, va, vml, vma, o_store, o_state);
    SP_ESTAMP(43);
    // the post-step scan (core.py:203-206); cos/sin of h1 == of wrap(h1)
    // (its dispatch prediction c.rec[e].qpred arrives by cp.async, see the kernel)
    add_slot(d, c, e, x, y, cos1, sin1, ep_sig, gid, ctr,
             r.ended && d.auto_reset ? -1 : (int32_t)s, o_store, o_state);
    ctr += d.nb;
    r.step_end = step;
    if (!r.handed) {
      d.x[s] = x; d.y[s] = y; d.h[s] = h; d.vl[s] = vl; d.va[s] = va;
      d.step[s] = step;
    }
    if (xs >= 0 && !late) {  // inline reset (no reset warp in this chunk)
      if (reset_env(d, mv, mc, s, gid, ctr, c, xs, a.states + row * d.D)) {
        c.xslot[e] = xs;
        c.wmode[e] = W_RESET_X;
      } else {
        set_error(d, SP_EMAP, row);
      }
    }
  }
  return r;
}

// The late auto-resets of a chunk (step_env with `late`), by the reset warp:
// once every env lane is past its reset decision, reset each handed-off env
// into its spare slot (SIMT across them; the hand-off -- env, stream
// position -- is parked in the slot's record), draw their scans' LiDAR noise,
// and list their (slot, group) entries right-aligned in the list's reserved
// prefix, just before the ordered entries -- while the other warps finish
// phase A and order the chunk's post-step scans.  So the ray queue starts
// with the fresh spawns (no step history: they rank longest).  ctl[22] =
// entries listed, ctl[23] = slots claimed; a failed spawn (SP_EMAP) gets
// hwrite -1 and no entries (its rows keep the post-step values).
__device__ __forceinline__ void reset_late(const EnvDev& d, const StepArgs& a, const MapView& mv,
                                           const MapConst& mc, const Chunk& c, int n, int64_t s0,
                                           uint64_t* bar, int map_par) {
  const int lane = threadIdx.x & 31;
  if (lane == 0)
    while (*(volatile int*)&c.ctl[21] < n) __nanosleep(64);
  __syncwarp();
  __threadfence_block();
  const int cap = d.chunk_cap;
  const int nres = min(*(volatile int*)&c.ctl[2], d.slot_cap - cap);
  if (nres > 0) {
    if (map_par >= 0) mbar_wait(bar, (uint32_t)map_par);
    for (int k = lane; k < nres; k += 32) {
      const int slot = cap + k;
      const int e = (int)c.rec[slot].qpred;
      uint64_t ctr = c.rec[slot].nctr;
      const int64_t s = s0 + e;
      const int64_t row = c.rowi[e];
      if (!reset_env(d, mv, mc, s, (uint32_t)(d.env_id_offset + row), ctr, c, slot,
                     a.states + row * d.D, false)) {
        set_error(d, SP_EMAP, row);
        c.hwrite[slot] = -1;
      }
      d.ctr[s] = ctr;
    }
    __syncwarp();
    // LiDAR noise of the reset scans (every slot's blocks over the warp)
    for (int it = lane; it < nres * d.nb; it += 32) {
      const int k = it / d.nb;
      if (c.hwrite[cap + k] >= 0) noise_block(d, c, cap + k, it - k * d.nb);
    }
  }
  // the spawned slots' entries, groups in order, ending at the reserved prefix
  const int G = d.n_groups;
  int good_n = 0;
  for (int k0 = 0; k0 < nres; k0 += 32)
    good_n += __popc(__ballot_sync(SP_FULL, k0 + lane < nres && c.hwrite[cap + k0 + lane] >= 0));
  uint16_t* dst = c.list + late_reserve(d) - good_n * G;
  int pos = 0;
  for (int k0 = 0; k0 < nres; k0 += 32) {
    const int k = k0 + lane;
    const bool good = k < nres && c.hwrite[cap + k] >= 0;
    const unsigned m = __ballot_sync(SP_FULL, good);
    if (good) {
      const int at = pos + __popc(m & lanemask_lt());
      for (int g = 0; g < G; ++g) dst[at * G + g] = (uint16_t)(((cap + k) << 3) | g);
    }
    pos += __popc(m);
  }
  if (lane == 0) {
    c.ctl[22] = good_n * G;
    c.ctl[23] = nres;
  }
}

// The per-env outputs and VecEnv statistics of one live env in MODE_STEP
// (vecenv.py:96-112), given the episode return before the step.  The reward
// is terminal (-10 / +75) or the shaped partial plus the proximity term from
// the env's scan, so collisions and arrivals finish in phase A and only
// running / timed-out envs wait for phase C.
__device__ __forceinline__ void finish_env(const EnvDev& d, const StepArgs& a, const Chunk& c,
                                           int e, int64_t s, int64_t row, int8_t ev,
                                           double partial, int32_t step_end, double ret_prev) {
  const double rew = ev == 1 ? -10.0
                   : ev == 2 ? 75.0
                             : dadd(partial, dmul(0.1, c.prox[e] ? -1.0 : 0.0));
  a.rewards[row] = rew;
  a.dones[row] = (uint8_t)(ev == 1 || ev == 2);
  a.truncated[row] = (uint8_t)(ev == 3);
  a.events[row] = ev;
  double ret = dadd(ret_prev, rew);  // vecenv.py:96-112
  if (ev != 0) {
    d.episodes[s] += 1;
    d.return_sum[s] = dadd(d.return_sum[s], ret);
    if (ev == 2) d.arrivals[s] += 1;
    const unsigned long long kk = atomicAdd(d.rec_count, 1ull);
    d.rec_ret[kk % d.rec_cap] = ret;
    d.rec_key[kk % d.rec_cap] = (a.step_index << 32) | (uint64_t)row;
    if (d.first_event[s] < 0) {
      d.first_event[s] = ev;
      d.first_ret[s] = ret;
      d.first_steps[s] = step_end;
    }
    ret = 0.0;
    if (!d.auto_reset || c.wmode[e] == W_RESET_OV) d.needs_reset[s] = 1;
  }
  d.ret[s] = ret;
}


// ------------------------------------------------------------ the kernel ---
template <bool kSmem, bool kRec>
__global__ void __launch_bounds__(SP_CTA_THREADS, SP_CTAS_PER_SM)
    env_step_kernel(const __grid_constant__ EnvDev d, const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  SP_STAMP(0);
#ifdef SP_TIMING
  if (threadIdx.x == 0) {  // CTA start on the GPU-wide clock (ns)
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)::"memory");
    s_sp_ts[36] = g;
  }
#endif
  double2* beam = (double2*)(smem + d.off_beam);
  uint64_t* bar = (uint64_t*)(smem + d.off_bar);
  const Chunk c = chunk_smem(smem, d);
  const bool plan = blockIdx.x < (unsigned)d.plan_n;
  // prologue: the beam table and the first map's constants, copied by
  // cp.async (one global round trip, no registers held)
  MapConst* smc = (MapConst*)(bar + 2);  // 72 B in the 128-B barrier block
  int smc_map = plan ? d.plan_map[blockIdx.x] : -1;
  for (int j = threadIdx.x; j < d.R; j += blockDim.x) {
    cp_async8(&beam[j].x, &d.beam_cs[j].x);
    cp_async8(&beam[j].y, &d.beam_cs[j].y);
  }
  if (plan && threadIdx.x < (int)(sizeof(MapConst) / 8))
    cp_async8((double*)smc + threadIdx.x, (const double*)(d.mconst + smc_map) + threadIdx.x);
  if (threadIdx.x == 0 && kSmem) mbar_init(bar, 1);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  SP_STAMP(1);
  uint32_t phase = 0;
  if (threadIdx.x == 0) bar[1] = (uint64_t)clock64();  // CTA start (kept in smem, not a register)
  const int64_t sb = plan ? d.plan_begin[blockIdx.x] : d.cta_begin[blockIdx.x];
  const int64_t se = plan ? d.plan_end[blockIdx.x] : d.cta_begin[blockIdx.x + 1];
  const int D = d.D;
  const FinObs<kRec> fin{c, D, d.max_range, d.inv_max_range, d.proximity, a.hit_store,
                         a.hit_state, a.scan_state, a.store_states,
                         (uint64_t)d.n * (uint64_t)D, (uint32_t)d.env_id_offset, d.R,
                         d.gshift, d.slot_cap};
  int m = plan ? d.plan_map[blockIdx.x] : 0, cur_map = -1;
  int64_t mstart = plan ? d.plan_mstart[blockIdx.x] : 0;  // map_off[m], map_off[m + 1]
  int64_t mend = plan ? d.plan_mend[blockIdx.x] : 0;
  int map_par = -1;  // parity of a map load not yet waited for, or -1
  // shared-memory tables always sit at the start of smem: seeding the view with
  // that address lets the march fold the table base into its LDS offsets
  MapView mv{};
  if constexpr (kSmem) {
    mv.blk = smem;
    mv.bits = (const uint32_t*)(smem + d.blk_bytes);
    mv.kbase = smem_u32(smem);
  }
  for (int64_t s0 = sb; s0 < se;) {
    if (!plan || s0 >= mend) {  // a further map (CTAs spanning maps): from the table
      while (d.map_off[m + 1] <= s0) ++m;
      mstart = d.map_off[m];
      mend = d.map_off[m + 1];
    }
    if (m != cur_map) {
      // the TMA lands while phase A loads its lanes; step_env waits right
      // before its first table read
      map_par = kSmem ? (int)phase : -1;
      mv = bind_map<kSmem>(d, m, smem, bar, phase, false);
      cur_map = m;
      SP_STAMP(2);
#ifdef SP_TIMING
      if (threadIdx.x == 0) {  // debug: this CTA's env count and map
        s_sp_ts[8] = (unsigned long long)(se - sb);
        s_sp_ts[9] = (unsigned long long)m;
      }
#endif
    }
    if (m != smc_map) {  // a further map (CTAs spanning maps): its constants
      __syncthreads();
      if (threadIdx.x < (int)(sizeof(MapConst) / 8))
        ((double*)smc)[threadIdx.x] = ((const double*)(d.mconst + m))[threadIdx.x];
      smc_map = m;
    }
    // the map's constants stay in shared memory, read where used: held in
    // registers across phase A they would cost 18 of the 80
    const MapConst& mc = *smc;
    const int n = (int)min((int64_t)d.chunk_cap, min(se, mend) - s0);
    const int e = threadIdx.x;
    const bool act = e < n;
    const int64_t s = s0 + e;
    const int64_t row = act ? row_of(d, m, mstart, s) : 0;
    const uint32_t gid = (uint32_t)(d.env_id_offset + row);
    // the lane's counter and action: loads in flight across the barrier below
    uint64_t ctr = act ? d.ctr[s] : 0;
    const int64_t av = act && a.mode == MODE_STEP ? a.actions[row] : 0;
    __syncthreads();  // the previous chunk is fully written out
    if (threadIdx.x < 4) c.ctl[threadIdx.x] = 0;
    if (threadIdx.x >= 21 && threadIdx.x < 24) c.ctl[threadIdx.x] = 0;
    // the warps without an env pre-noise the first kpre env slots during phase
    // A, d.prenoise blocks per thread (what fits in phase A's latency: more
    // would make them its tail); every thread does the rest after phase A.
    // Only whole idle warps: a warp mixing env and noise threads runs both
    // paths one after the other and became phase A's slowest warp
    const int first_idle = (n + 31) & ~31;
    // late resets: the first warp without an env becomes the reset warp
    // (reset_late) when another idle warp is left for the pre-noise; the other
    // warps then run phase A's end and the ordering on barrier 2 without it
    const bool late = a.mode == MODE_STEP && d.auto_reset && d.late_resets &&
                      (int)blockDim.x - first_idle >= 64;
    const int first_pre = first_idle + (late ? 32 : 0);
    const bool rw = late && e >= first_idle && e < first_pre;
    const int kpre = a.mode == MODE_STEP
                         ? min(n, d.prenoise * max(0, (int)blockDim.x - first_pre) / d.nb)
                         : 0;
    if (act) c.rowi[e] = (int32_t)row;
    if (act && a.mode == MODE_STEP) {
      // copied without registers, waited for where used: the post-step scan's
      // step history (before the ray order) and the episode constants phase A
      // needs late, parked in this env's scan-slot words until add_slot
      // overwrites them (cross-track start, obs-header start heading, sigma)
      cp_async8(&c.rec[e].qpred, &d.qhist[s]);
      cp_async8(&c.rec[e].px, d.sx + s);
      cp_async8(&c.rec[e].py, d.sy + s);
      cp_async8(&c.rec[e].ch, d.c0 + s);
      cp_async8(&c.rec[e].sh, d.s0 + s);
      cp_async8(&c.rec[e].sig, d.psig + s);
    }
    __syncthreads();
    if (kpre > 0 && e >= first_pre) prenoise(d, a, c, kpre, first_pre, s0, m, mstart);
    if (rw) reset_late(d, a, mv, mc, c, n, s0, bar, map_par);

    // ---- A: physics, collision, events, reward partial, resets -----------
    if (act) {
      c.xslot[e] = -1;
      c.wmode[e] = W_NONE;
      c.evs[e] = -1;
    }
    if (a.mode != MODE_STEP) {
      const bool want = a.mode == MODE_RESET_ALL || (act && a.reset_mask[row] != 0);
      if (map_par >= 0) mbar_wait(bar, (uint32_t)map_par);
      if (act && want) {
        if (reset_env(d, mv, mc, s, gid, ctr, c, e, a.states + row * d.D)) {
          c.wmode[e] = W_STATE;
          if (a.mode == MODE_RESET_ALL) {
            d.ret[s] = 0.0;
            d.first_event[s] = -1;
          }
        } else {
          set_error(d, SP_EMAP, row);
        }
        d.ctr[s] = ctr;
      }
    } else if (act) {
      const double ret_prev = d.ret[s];  // issued early: only the outputs wait on it
      const StepA r = step_env(d, a, mv, mc, c, e, s, row, gid, ctr, av, d.chunk_cap, d.slot_cap,
                               bar, map_par, late);
      if (!r.handed) d.ctr[s] = ctr;
      if (r.live) {
        if (r.ev == 1 || r.ev == 2) {  // terminal reward: no scan needed
          finish_env(d, a, c, e, s, row, r.ev, 0.0, r.step_end, ret_prev);
        } else {
          c.evs[e] = r.ev;
          c.part[e] = r.partial;
          c.send[e] = r.step_end;
          c.retp[e] = ret_prev;
        }
      }
    }
    if (map_par >= 0) {  // threads without an env have not waited for the tables yet
      mbar_wait(bar, (uint32_t)map_par);
      map_par = -1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef SP_TIMING
    if ((threadIdx.x & 31) == 0) {  // each warp's arrival (lane 0) at the end of phase A
      unsigned long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
      s_sp_ts[12 + (threadIdx.x >> 5)] = t;
    }
#endif
    // ---- N: LiDAR noise + longest-first ray order; B: LiDAR rays ------------
    // (all threads but the reset warp, which joins at the ray phase)
    const int reserve = late ? late_reserve(d) : 0;
    if (!rw) {
      const Grp main = late ? Grp{(int)threadIdx.x - (e >= first_pre ? 32 : 0), (int)blockDim.x - 32, 2}
                            : cta_grp();
      main.sync();
      SP_STAMP(3);
      const int n_main = c.ctl[1];
      order_entries(d, c, n_main, main, c.list + reserve);
      SP_STAMP(11);
      SP_WSTAMP(48);
      noise_phase(d, c, n_main, kpre, main);
    }
    __syncthreads();
    SP_STAMP(4);
    SP_WSTAMP(72);
    const int n_slots = c.ctl[1];
    const int n_late = c.ctl[22];  // late-reset entries, right before the ordered ones
    ray_phase<kSmem, kRec>(mv, d, c, beam, c.list + reserve - n_late, c.ctl[20] + n_late, fin);
    SP_WSTAMP(96);
    __syncthreads();
    SP_STAMP(5);
    store_history(d, c, n_slots, c.ctl[23]);
    // ---- C: reward, outputs, statistics of running / timed-out envs --------
    if (act && c.evs[e] >= 0)
      finish_env(d, a, c, e, s, c.rowi[e], c.evs[e], c.part[e], c.send[e], c.retp[e]);
    SP_STAMP(6);
    // ---- overflow pass: resets that did not fit the extra slots (rare) -----
    if (a.mode == MODE_STEP && c.ctl[3] > 0) {
      __syncthreads();
      if (threadIdx.x < 2) c.ctl[threadIdx.x] = 0;
      __syncthreads();
      if (act && c.wmode[e] == W_RESET_OV) {
        uint64_t ctr2 = d.ctr[s];
        const int64_t row2 = c.rowi[e];
        if (reset_env(d, mv, mc, s, (uint32_t)(d.env_id_offset + row2), ctr2, c, e,
                      a.states + row2 * d.D)) {
          c.wmode[e] = W_STATE;
        } else {
          set_error(d, SP_EMAP, row2);
          c.wmode[e] = W_NONE;
        }
        d.ctr[s] = ctr2;
      } else if (act) {
        c.wmode[e] = W_NONE;
      }
      __syncthreads();
      const int n2 = c.ctl[1];
      order_entries(d, c, n2, cta_grp(), c.list);
      noise_phase(d, c, n2, 0, cta_grp());
      __syncthreads();
      ray_phase<kSmem, kRec>(mv, d, c, beam, c.list, c.ctl[20], fin);
      __syncthreads();
      store_history(d, c, n2);
    }
    SP_STAMP(7);
    s0 += n;
  }
#ifdef SP_TIMING
  sp_stamp_flush();
#endif
  if (a.mode == MODE_STEP) {  // per-CTA duration (launch diagnostics: sp_env_launch_info)
    __syncthreads();
    if (threadIdx.x == 0)
      d.cta_cyc[blockIdx.x] = (uint32_t)min(clock64() - (long long)bar[1], (long long)UINT32_MAX);
  }
}

// Standalone LiDAR scan on caller poses (cfg4): the same marcher, no noise.
struct FinScan {
  double* ranges;
  int32_t* hit_cell;
  int64_t s0;
  int R;
  __device__ __forceinline__ float pre(int, int) const { return 0.0f; }
  __device__ __forceinline__ void operator()(int e, int j, double t, int hit, int, float) const {
    const int64_t o = (s0 + e) * R + j;
    ranges[o] = t;
    if (hit_cell) hit_cell[o] = hit;
  }
};

#ifndef SP_SCAN_THREADS
#define SP_SCAN_THREADS SP_CTA_THREADS
#endif
template <bool kSmem>
__global__ void __launch_bounds__(SP_SCAN_THREADS, SP_CTAS_PER_SM)
    env_scan_kernel(const __grid_constant__ EnvDev d, const __grid_constant__ ScanArgs q) {
  extern __shared__ __align__(128) uint8_t smem[];
  double2* beam = (double2*)(smem + d.off_beam);
  uint64_t* bar = (uint64_t*)(smem + d.off_bar);
  const Chunk c = chunk_smem(smem, d);
  for (int j = threadIdx.x; j < d.R; j += blockDim.x) beam[j] = d.beam_cs[j];
  if (threadIdx.x == 0 && kSmem) mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  const int64_t sb = q.cta_begin[blockIdx.x], se = q.cta_begin[blockIdx.x + 1];
  int m = 0, cur_map = -1;
  // shared-memory tables always sit at the start of smem: seeding the view with
  // that address lets the march fold the table base into its LDS offsets
  MapView mv{};
  if constexpr (kSmem) {
    mv.blk = smem;
    mv.bits = (const uint32_t*)(smem + d.blk_bytes);
    mv.kbase = smem_u32(smem);
  }
  for (int64_t s0 = sb; s0 < se;) {
    while (q.qoff[m + 1] <= s0) ++m;
    if (m != cur_map) {
      mv = bind_map<kSmem>(d, m, smem, bar, phase);
      cur_map = m;
    }
    const int n = (int)min((int64_t)d.chunk_cap, min(se, q.qoff[m + 1]) - s0);
    __syncthreads();
    if (threadIdx.x == 0) {
      c.ctl[0] = 0;
      c.ctl[20] = n * d.n_groups;  // entries listed (the order is the query order)
    }
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      double sh_, ch_;
      sincos(q.h[s0 + e], &sh_, &ch_);
      c.rec[e].px = q.x[s0 + e];
      c.rec[e].py = q.y[s0 + e];
      c.rec[e].ch = ch_;
      c.rec[e].sh = sh_;
      for (int g = 0; g < d.n_groups; ++g) c.list[e * d.n_groups + g] = (uint16_t)((e << 3) | g);
    }
    __syncthreads();
    const FinScan fin{q.ranges, q.hit_cell, s0, d.R};
    ray_phase<kSmem, true>(mv, d, c, beam, c.list, n * d.n_groups, fin);
    s0 += n;
  }
}


}  // namespace sp

