// sp_ops.cu -- op-level plugin kernels, the replay ring, benchmark helpers.
//
// * cast_rays_exact / disc_collides: the reference kernel seam
//   (kernels/__init__.py:62-86) on device.  cast_rays_exact restates the
//   reference algorithm itself (DDA + EDT jump, _cy.pyx:19-106) operation for
//   operation in IEEE fp64 without contraction, so it is bit-identical to the
//   Cython backend on any occupancy grid -- including grids without an
//   occupied border, where the reference's jump may land outside the grid and
//   report the landing distance.  Lane per ray; occ/edt read through L1/L2.
// * Replay ring (replay.py:31-87): append = contiguous ring writes (the ring
//   rows are contiguous, so a batch is one flat wrapped copy per column);
//   sample = Philox index draw (replay.py:76) + row gather.
#include "sp_common.cuh"

namespace sp {

__global__ void cast_rays_exact_kernel(const uint8_t* __restrict__ occ,
                                       const double* __restrict__ edt, int64_t H, int64_t W,
                                       const int64_t* __restrict__ map_idx,
                                       const double* __restrict__ px,
                                       const double* __restrict__ py,
                                       const double* __restrict__ dirx,
                                       const double* __restrict__ diry, int64_t n, double cell,
                                       double max_range, double* __restrict__ out) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = map_idx[r];
    const uint8_t* o = occ + m * H * W;
    const double* e = edt + m * H * W;
    const double x0 = px[r], y0 = py[r], dx = dirx[r], dy = diry[r];
    int64_t ix = (int64_t)floor(ddiv(x0, cell));
    int64_t iy = (int64_t)floor(ddiv(y0, cell));
    if (ix < 0 || ix >= W || iy < 0 || iy >= H || o[iy * W + ix]) {  // :37-42
      out[r] = 0.0;
      continue;
    }
    const int64_t stepx = dx > 0 ? 1 : (dx < 0 ? -1 : 0);
    const int64_t stepy = dy > 0 ? 1 : (dy < 0 ? -1 : 0);
    const double tdx = dx != 0 ? ddiv(cell, fabs(dx)) : INF;
    const double tdy = dy != 0 ? ddiv(cell, fabs(dy)) : INF;
    double tmx = dx > 0 ? ddiv(dsub(dmul((double)(ix + 1), cell), x0), dx)
                        : (dx < 0 ? ddiv(dsub(dmul((double)ix, cell), x0), dx) : INF);
    double tmy = dy > 0 ? ddiv(dsub(dmul((double)(iy + 1), cell), y0), dy)
                        : (dy < 0 ? ddiv(dsub(dmul((double)iy, cell), y0), dy) : INF);
    double t = 0.0, res = max_range;
    for (;;) {
      const double clearance = e[iy * W + ix];
      if (clearance > 2.5) {  // EDT jump, :62-88
        const double tj = dadd(t, dmul(dsub(clearance, 1.5), cell));
        const double qx = dadd(x0, dmul(tj, dx));
        const double qy = dadd(y0, dmul(tj, dy));
        ix = (int64_t)floor(ddiv(qx, cell));
        iy = (int64_t)floor(ddiv(qy, cell));
        tmx = dx > 0 ? dadd(ddiv(dsub(dmul((double)(ix + 1), cell), qx), dx), tj)
                     : (dx < 0 ? dadd(ddiv(dsub(dmul((double)ix, cell), qx), dx), tj) : INF);
        tmy = dy > 0 ? dadd(ddiv(dsub(dmul((double)(iy + 1), cell), qy), dy), tj)
                     : (dy < 0 ? dadd(ddiv(dsub(dmul((double)iy, cell), qy), dy), tj) : INF);
        t = tj;
        if (t > max_range) { res = max_range; break; }
        if (ix < 0 || ix >= W || iy < 0 || iy >= H) { res = t < max_range ? t : max_range; break; }
        continue;
      }
      if (tmx <= tmy) {  // :89-96
        t = tmx;
        tmx = dadd(tmx, tdx);
        ix += stepx;
      } else {
        t = tmy;
        tmy = dadd(tmy, tdy);
        iy += stepy;
      }
      if (t > max_range) { res = max_range; break; }
      if (ix < 0 || ix >= W || iy < 0 || iy >= H) { res = t < max_range ? t : max_range; break; }
      if (o[iy * W + ix]) { res = t < max_range ? t : max_range; break; }
    }
    out[r] = res;
  }
}

__global__ void disc_collides_kernel(const uint8_t* __restrict__ occ, int64_t H, int64_t W,
                                     const int64_t* __restrict__ map_idx,
                                     const double* __restrict__ px, const double* __restrict__ py,
                                     const double* __restrict__ radius, int64_t n, double cell,
                                     uint8_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double x = px[k], y = py[k], r = radius[k];
    if (x - r < 0.0 || y - r < 0.0 || x + r > (double)W * cell || y + r > (double)H * cell) {
      out[k] = 1;  // :124-126
      continue;
    }
    const uint8_t* o = occ + map_idx[k] * H * W;
    int64_t ix0 = (int64_t)floor(ddiv(dsub(x, r), cell)); if (ix0 < 0) ix0 = 0;
    int64_t ix1 = (int64_t)floor(ddiv(dadd(x, r), cell)); if (ix1 > W - 1) ix1 = W - 1;
    int64_t iy0 = (int64_t)floor(ddiv(dsub(y, r), cell)); if (iy0 < 0) iy0 = 0;
    int64_t iy1 = (int64_t)floor(ddiv(dadd(y, r), cell)); if (iy1 > H - 1) iy1 = H - 1;
    const double r2 = dmul(r, r);
    uint8_t hit = 0;
    for (int64_t iy = iy0; iy <= iy1 && !hit; ++iy) {
      for (int64_t ix = ix0; ix <= ix1; ++ix) {
        if (!o[iy * W + ix]) continue;
        double lo = dmul((double)ix, cell), hi = dadd(lo, cell);
        double nx = x > lo ? x : lo;
        if (nx > hi) nx = hi;
        lo = dmul((double)iy, cell);
        hi = dadd(lo, cell);
        double ny = y > lo ? y : lo;
        if (ny > hi) ny = hi;
        const double ddx = dsub(x, nx), ddy = dsub(y, ny);
        if (dadd(dmul(ddx, ddx), dmul(ddy, ddy)) <= r2) { hit = 1; break; }
      }
    }
    out[k] = hit;
  }
}

// ---------------------------------------------------------------- replay ---
// Ring append (replay.py:48-67): the n new rows land at rows cursor .. and
// wrap to 0, so every column is at most two contiguous segments.  The state
// columns s, s2 are row-contiguous float32 (D per row): four flat float
// segments (s and s2, before and after the wrap).  Each segment is a head of
// <= 3 floats (up to the first 16-byte aligned ring address), a body of
// float4 stores and a tail of <= 3 floats.  The bodies of all four segments
// form one index space that every thread walks kAppendU vectors at a time,
// all loads issued before any store (sources read as float4 when equally
// aligned -- always when the cursor is a multiple of 4 rows -- else as four
// coalesced scalars), so a launch is one HBM round trip deep.  The small
// columns (a i64, r f32, done u8: 13 B/row) follow the same pattern.
constexpr int kAppendU = 4;

struct AppendSeg {
  float* dst[4];
  const float* src[4];
  int64_t head[4];   // floats before the aligned body
  int64_t nvec[4];   // float4 body vectors
  int64_t count[4];  // floats in the segment
  int64_t vend[4];   // inclusive prefix sums of nvec
  int nseg;
};

__device__ __forceinline__ float4 load4(const float* p) {
  if (((uintptr_t)p & 15) == 0) return __ldcs((const float4*)p);
  return make_float4(__ldcs(p), __ldcs(p + 1), __ldcs(p + 2), __ldcs(p + 3));
}

__global__ void __launch_bounds__(256) rb_append_kernel(
    const __grid_constant__ AppendSeg g, int64_t* __restrict__ ra, float* __restrict__ rr,
    uint8_t* __restrict__ rd, int64_t cap, int64_t cursor, const int64_t* __restrict__ a,
    const void* __restrict__ r, int r_f64, const uint8_t* __restrict__ dn, int64_t n,
    int64_t* __restrict__ d_size, int64_t new_size) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  if (t == 0) *d_size = new_size;  // the ring's fill, on device (sp_rb_sample_dev)
  // heads and tails: <= 6 scalars per segment
  if (t < 6 * g.nseg) {
    const int k = (int)(t / 6), e = (int)(t % 6);
    const int64_t i = e < 3 ? e : g.head[k] + 4 * g.nvec[k] + (e - 3);
    if ((e < 3 && i < g.head[k]) || (e >= 3 && i < g.count[k])) g.dst[k][i] = g.src[k][i];
  }
  const int64_t total = g.vend[g.nseg - 1];
  for (int64_t base = t; base < total; base += kAppendU * nt) {
    float4 v[kAppendU];
    float4* dp[kAppendU];
#pragma unroll
    for (int u = 0; u < kAppendU; ++u) {
      const int64_t q = base + u * nt;
      dp[u] = nullptr;
      if (q < total) {
        int k = 0;
        while (q >= g.vend[k]) ++k;
        const int64_t j = q - (k ? g.vend[k - 1] : 0);
        const int64_t off = g.head[k] + 4 * j;
        v[u] = load4(g.src[k] + off);
        dp[u] = (float4*)(g.dst[k] + off);
      }
    }
#pragma unroll
    for (int u = 0; u < kAppendU; ++u)
      if (dp[u]) *dp[u] = v[u];
  }
  const int64_t n1 = n < cap - cursor ? n : cap - cursor;  // rows before the wrap
  for (int64_t base = t; base < n; base += kAppendU * nt) {
    int64_t av[kAppendU];
    float rv[kAppendU];
    uint8_t dv[kAppendU];
#pragma unroll
    for (int u = 0; u < kAppendU; ++u) {
      const int64_t i = base + u * nt;
      if (i < n) {
        av[u] = a[i];
        rv[u] = r_f64 ? (float)((const double*)r)[i] : ((const float*)r)[i];  // replay.py:53
        dv[u] = dn[i] ? 1 : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < kAppendU; ++u) {
      const int64_t i = base + u * nt;
      if (i < n) {
        const int64_t row = i < n1 ? cursor + i : i - n1;
        ra[row] = av[u];
        rr[row] = rv[u];
        rd[row] = dv[u];
      }
    }
  }
}

// One warp per sampled row (8 rows per CTA): every lane draws the row's index
// (Philox block ctr + i of (seed, stream_id, tag 2), replay.py:76), then the
// lanes copy its columns coalesced.  All rows' random ring reads are in flight
// at once instead of one thread walking a row serially.
// d_size / d_ctr (nullable): read the fill and the first Philox block from
// device memory instead (sp_rb_sample_dev: graph-capturable sampling).
__global__ void rb_sample_kernel(const float* __restrict__ rs, const int64_t* __restrict__ ra,
                                 const float* __restrict__ rr, const float* __restrict__ rs2,
                                 const uint8_t* __restrict__ rd, int32_t dim, int64_t size,
                                 int64_t batch, uint64_t seed, uint32_t stream_id, uint64_t ctr,
                                 float* __restrict__ s, int64_t* __restrict__ a,
                                 float* __restrict__ r, float* __restrict__ s2,
                                 uint8_t* __restrict__ dn, int64_t* __restrict__ idx_out,
                                 const int64_t* __restrict__ d_size,
                                 const uint64_t* __restrict__ d_ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= batch) return;
  if (d_size) size = *d_size;
  if (d_ctr) ctr = *d_ctr;
  if (size < 1) return;  // nothing stored (the caller gates on its host-side size)
  const Block4 b = stream_block(seed, stream_id, 2u, ctr + (uint64_t)i);
  const int64_t k = draw_integer(b, 0, size);
  if (lane == 0) {
    a[i] = ra[k];
    r[i] = rr[k];
    dn[i] = rd[k];
    if (idx_out) idx_out[i] = k;
  }
  const float* src = rs + k * dim;
  const float* src2 = rs2 + k * dim;
  float* dst = s + i * dim;
  float* dst2 = s2 + i * dim;
  int c = lane;
  for (; c + 32 < dim; c += 64) {  // both rows' loads in flight before the stores
    const float v0 = src[c], v1 = src[c + 32], w0 = src2[c], w1 = src2[c + 32];
    dst[c] = v0; dst[c + 32] = v1; dst2[c] = w0; dst2[c + 32] = w1;
  }
  if (c < dim) {
    const float v0 = src[c], w0 = src2[c];
    dst[c] = v0;
    dst2[c] = w0;
  }
}

__global__ void rb_ctr_advance_kernel(uint64_t* ctr, int64_t n) { *ctr += (uint64_t)n; }

__global__ void rb_gather_kernel(const float* __restrict__ rs, const int64_t* __restrict__ ra,
                                 const float* __restrict__ rr, const float* __restrict__ rs2,
                                 const uint8_t* __restrict__ rd, int32_t dim, int64_t size,
                                 float* __restrict__ s, int64_t* __restrict__ a,
                                 float* __restrict__ r, float* __restrict__ s2,
                                 uint8_t* __restrict__ dn) {
  const int64_t flat = size * dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < flat;
       i += (int64_t)gridDim.x * blockDim.x) {
    s[i] = rs[i];
    s2[i] = rs2[i];
    if (i < size) {
      a[i] = ra[i];
      r[i] = rr[i];
      dn[i] = rd[i];
    }
  }
}

// --------------------------------------------------------------- bench ----
__global__ void random_actions_kernel(int64_t n, uint64_t seed, int64_t env_id0, int64_t step,
                                      int32_t n_actions, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Block4 b = stream_block(seed, (uint32_t)(env_id0 + i), 1u, (uint64_t)step);
    out[i] = draw_integer(b, 0, n_actions);
  }
}

__global__ void philox_fill_kernel(int64_t n, uint64_t seed, uint32_t lane, uint32_t tag,
                                   uint64_t ctr0, int kind, double lo, double hi, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Block4 b = stream_block(seed, lane, tag, ctr0 + (uint64_t)i);
    if (kind == 0)
      ((double*)out)[i] = draw_uniform(b, lo, hi);
    else
      ((int64_t*)out)[i] = draw_integer(b, (int64_t)lo, (int64_t)hi);
  }
}

// Lanes whose first episode has not ended yet (first_event < 0), into *out.
__global__ void count_pending_kernel(const int8_t* __restrict__ first_event, int64_t n,
                                     unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += first_event[i] < 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(SP_FULL, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Deterministic single-CTA totals {episodes, arrivals, return_sum}.
__global__ void stats_totals_kernel(const int64_t* __restrict__ eps,
                                    const int64_t* __restrict__ arr,
                                    const double* __restrict__ rsum, int64_t n,
                                    double* __restrict__ out3) {
  __shared__ double se[1024], sa[1024], sr[1024];
  double e = 0, a = 0, r = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    e += (double)eps[i];
    a += (double)arr[i];
    r += rsum[i];
  }
  se[threadIdx.x] = e;
  sa[threadIdx.x] = a;
  sr[threadIdx.x] = r;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      se[threadIdx.x] += se[threadIdx.x + w];
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sr[threadIdx.x] += sr[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out3[0] = se[0];
    out3[1] = sa[0];
    out3[2] = sr[0];
  }
}

// Bias-corrected Adam over up to SP_ADAM_MAX tensors in one launch
// (net.py:141-161), with the reference's operation order and fp32 roundings:
//   m = m*b1 + (1-b1)*g;  v = v*b2 + (1-b2)*g^2;
//   p -= (lr * (m / c1)) / (sqrt(v / c2) + eps),  c_k = f32(1 - beta_k^t) in f64.
// Python-double scalars are rounded to f32 as numpy's weak-scalar rule does.
// gate (nullable): apply only if *gate is finite (ddqn.py:66-71 abort leaves
// the state untouched). t = step_dev ? *step_dev + 1 : step_host.
struct AdamTensors {
  float* p[SP_ADAM_MAX];
  const float* g[SP_ADAM_MAX];
  float* m[SP_ADAM_MAX];
  float* v[SP_ADAM_MAX];
  int64_t end[SP_ADAM_MAX];  // inclusive prefix sums of numels
  int n;
};

__global__ void adam_kernel(const __grid_constant__ AdamTensors T, const double* step_dev,
                            int64_t step_host, const float* gate, double lr, double b1,
                            double b2, double eps) {
  if (gate && !isfinite(*gate)) return;
  const double t = step_dev ? *step_dev + 1.0 : (double)step_host;
  const float c1 = (float)(1.0 - pow(b1, t));
  const float c2 = (float)(1.0 - pow(b2, t));
  const float fb1 = (float)b1, fb2 = (float)b2, f1b1 = (float)(1.0 - b1),
              f1b2 = (float)(1.0 - b2), flr = (float)lr, feps = (float)eps;
  const int64_t total = T.end[T.n - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    while (i >= T.end[k]) ++k;
    const int64_t j = i - (k ? T.end[k - 1] : 0);
    const float g = T.g[k][j];
    const float m = __fadd_rn(__fmul_rn(T.m[k][j], fb1), __fmul_rn(f1b1, g));
    const float v = __fadd_rn(__fmul_rn(T.v[k][j], fb2), __fmul_rn(f1b2, __fmul_rn(g, g)));
    T.m[k][j] = m;
    T.v[k][j] = v;
    const float m_hat = __fdiv_rn(m, c1);
    const float v_hat = __fdiv_rn(v, c2);
    const float upd = __fdiv_rn(__fmul_rn(flr, m_hat), __fadd_rn(__fsqrt_rn(v_hat), feps));
    T.p[k][j] = __fsub_rn(T.p[k][j], upd);
  }
}

__global__ void adam_tick_kernel(double* step_dev, const float* gate) {
  if (!gate || isfinite(*gate)) *step_dev += 1.0;
}

}  // namespace sp
