// sp_actor.cu -- the actor's half of an ASL iteration in one launch (SURVEY
// 8(f) row 1; the reference's asl/loops.py:57-60):
//
//   q       = MLP(states)                 net.py:63-80 ([D0, H1, H2, A], ReLU)
//   eps_i   = VEM epsilon of copy i at t_step   asl/vem.py:38-54
//   action  = random action with prob eps_i, else argmax_j q[i, j]
//                                         asl/vem.py:57-66
//
// Draws follow the Philox contract (sp_philox_fill, asl.select_actions): row
// i's explore test uses block ctr + i (uniform), its random action block
// ctr + n + i (integers(0, A)), as the reference's random(n) then
// integers(0, A, n); the caller advances its stream by 2 n.  The epsilon is
// computed on the device from the scalar t_step in the reference's float64
// operation order, so no per-step host array exists.
//
// Layout: a persistent CTA per SM stages the three weight matrices into
// shared memory once (TMA bulk copies) and walks tiles of `rows` rows (32
// when the weights leave room), the next tile's states loaded into registers
// while this one computes.  The dense layers are fp32 FMA in k-ascending
// order (the fused learner's order; last-bit differences from BLAS blocking
// only), register-blocked 8 rows x 4 columns per thread with the column
// pairs on FFMA2 (two fp32 FMAs per instruction, each rounded as fmaf), so a
// weight quad loaded from shared memory -- the traffic that bounds the loop
// -- feeds 32 FMAs.  A sum then adds the bias (x @ W + b, net.py:63-74).
// tools/bench_actor.py at 65,536 rows: 281 us (4 x 4 blocks, one FFMA per
// multiply-add) -> 236 us (FFMA2, 16-byte x loads) -> 220 us (8 x 4 blocks).
#pragma once
#include "sp_common.cuh"

namespace sp {

constexpr int kActThreads = 256;
constexpr int kActMaxD0 = 64, kActMaxH = 256, kActMaxA = 16;
constexpr int kActPre = 8;  // prefetched state floats per thread: TR * pad4(D0) <= 8 * 256

struct VemDev {
  int64_t n_envs, or_init, or_final, decay_steps;
  double e_min, e_max;
};

struct ActorArgs {
  const float* W[3];
  const float* b[3];
  int D0, H1, H2, A, L0;  // L0 = pad4(D0): the staged state row stride
  int rows;               // rows per tile
  const float* states;    // (n, D0)
  int64_t n;
  int64_t env0;           // VEM copy index of row 0 (env id offset of a shard)
  VemDev vem;
  int64_t t_step;
  uint64_t seed;
  uint32_t lane, tag;
  uint64_t ctr;
  int64_t* actions;       // (n,)
  float* q_out;           // (n, A) or null: the Q-values (tests, evaluation)
};

// vem.py:38-40 exploring_interval, then :42-54 epsilon(i), float64 ops in the
// reference's order (the explore test compares against it bit for bit)
// the exploring interval's size at t_step (row-independent)
__device__ __forceinline__ int64_t vem_size(const VemDev& v, int64_t t_step) {
  double frac = __ddiv_rn((double)t_step, (double)v.decay_steps);
  if (frac > 1.0) frac = 1.0;
  const double span = __dmul_rn((double)(v.or_final - v.or_init), frac);
  return (int64_t)floor(__dadd_rn(__dadd_rn((double)v.or_init, span), 0.5));
}
__device__ __forceinline__ double vem_epsilon_sized(const VemDev& v, int64_t i, int64_t size) {
  const int64_t first = v.n_envs - size;
  if (i < first) return v.e_min;
  if (i == v.n_envs - 1) return v.e_max;  // ramp top, exact endpoint
  return __dadd_rn(v.e_min, __ddiv_rn(__dmul_rn(__dsub_rn(v.e_max, v.e_min), (double)(i - first)),
                                      (double)(size - 1)));
}
__device__ __forceinline__ double vem_epsilon(const VemDev& v, int64_t i, int64_t t_step) {
  const int64_t size = vem_size(v, t_step);
  const int64_t first = v.n_envs - size;
  if (i < first) return v.e_min;
  if (i == v.n_envs - 1) return v.e_max;  // ramp top, exact endpoint
  return __dadd_rn(v.e_min, __ddiv_rn(__dmul_rn(__dsub_rn(v.e_max, v.e_min), (double)(i - first)),
                                      (double)(size - 1)));
}

// y[r][j] = act(b[j] + sum_k x[r][k] W[k][j]) for the tile's `rows` rows,
// 8 x 4 or 4 x 4 register blocks when n_out % 4 == 0, else one thread per output
__device__ __forceinline__ void act_dense(const float* x, int ldx, int n_in, const float* W,
                                          const float* b, int n_out, float* y, int rows,
                                          bool relu) {
#ifndef SP_ACTOR_4X4
  if ((n_out & 3) == 0 && (rows & 7) == 0 && (ldx & 3) == 0) {
    // 8 rows x 4 columns per thread: a warp's lanes hold consecutive column
    // quads of the same 8 rows, so each k's weight quad (the shared-memory
    // traffic that bounds this loop: 4 wavefronts per warp and k) feeds twice
    // the FMAs of a 4 x 4 block; x comes as 16-byte k-quads (a broadcast).
    // Same k-ascending fmaf chain per output (FFMA2 pairs).
    const int cq = n_out >> 2, tiles = (rows >> 3) * cq;
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
      const int rq = t / cq, jq = t - rq * cq;
      const float* xr = x + (rq * 8) * ldx;
      const float* wc = W + 4 * jq;
      float2 a2[8][2];
#pragma unroll
      for (int r = 0; r < 8; ++r) a2[r][0] = a2[r][1] = make_float2(0.0f, 0.0f);
      const int k4 = n_in & ~3;
      for (int k0 = 0; k0 < k4; k0 += 4) {
        float4 w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = *(const float4*)(wc + (k0 + i) * n_out);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float4 xv = *(const float4*)(xr + r * ldx + k0);
          const float xk[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            a2[r][0] = __ffma2_rn(make_float2(xk[i], xk[i]), make_float2(w[i].x, w[i].y), a2[r][0]);
            a2[r][1] = __ffma2_rn(make_float2(xk[i], xk[i]), make_float2(w[i].z, w[i].w), a2[r][1]);
          }
        }
      }
      for (int k = k4; k < n_in; ++k) {
        const float4 w = *(const float4*)(wc + k * n_out);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float xk = xr[r * ldx + k];
          a2[r][0] = __ffma2_rn(make_float2(xk, xk), make_float2(w.x, w.y), a2[r][0]);
          a2[r][1] = __ffma2_rn(make_float2(xk, xk), make_float2(w.z, w.w), a2[r][1]);
        }
      }
      const float4 bb = *(const float4*)(b + 4 * jq);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float o[4] = {__fadd_rn(a2[r][0].x, bb.x), __fadd_rn(a2[r][0].y, bb.y),
                      __fadd_rn(a2[r][1].x, bb.z), __fadd_rn(a2[r][1].y, bb.w)};
        if (relu)
#pragma unroll
          for (int c = 0; c < 4; ++c) o[c] = o[c] < 0.0f ? 0.0f : o[c];  // NaN stays NaN
        *(float4*)(y + (rq * 8 + r) * n_out + 4 * jq) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    return;
  }
#endif
  if ((n_out & 3) == 0 && (rows & 3) == 0) {
    const int cq = n_out >> 2, tiles = (rows >> 2) * cq;
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
      const int rq = t / cq, jq = t - rq * cq;
      float acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0f;
      const float* xr = x + (rq * 4) * ldx;
#ifdef SP_ACTOR_SCALAR  // reference form (A/B): one FFMA per multiply-add
      for (int k = 0; k < n_in; ++k) {
        const float4 w = *(const float4*)(W + k * n_out + 4 * jq);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float xv = xr[r * ldx + k];
          acc[r][0] = fmaf(xv, w.x, acc[r][0]);
          acc[r][1] = fmaf(xv, w.y, acc[r][1]);
          acc[r][2] = fmaf(xv, w.z, acc[r][2]);
          acc[r][3] = fmaf(xv, w.w, acc[r][3]);
        }
      }
#else
      // four k per trip: each row's x[k..k+3] is one 16-byte load (ldx and
      // the rows are 16-byte aligned), and the column pairs go through
      // FFMA2 (two independent fp32 FMAs, each rounded as fmaf): the same
      // k-ascending fmaf chain per output, half the FMA instructions and a
      // quarter of the x loads
      float2 a2[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) a2[r][0] = a2[r][1] = make_float2(0.0f, 0.0f);
      const int k4 = (ldx & 3) == 0 ? (n_in & ~3) : 0;  // unaligned rows: the one-k loop
      for (int k0 = 0; k0 < k4; k0 += 4) {
        float4 xv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) xv[r] = *(const float4*)(xr + r * ldx + k0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 w = *(const float4*)(W + (k0 + i) * n_out + 4 * jq);
          const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float xk = i == 0 ? xv[r].x : i == 1 ? xv[r].y : i == 2 ? xv[r].z : xv[r].w;
            a2[r][0] = __ffma2_rn(make_float2(xk, xk), w01, a2[r][0]);
            a2[r][1] = __ffma2_rn(make_float2(xk, xk), w23, a2[r][1]);
          }
        }
      }
      for (int k = k4; k < n_in; ++k) {
        const float4 w = *(const float4*)(W + k * n_out + 4 * jq);
        const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float xk = xr[r * ldx + k];
          a2[r][0] = __ffma2_rn(make_float2(xk, xk), w01, a2[r][0]);
          a2[r][1] = __ffma2_rn(make_float2(xk, xk), w23, a2[r][1]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[r][0] = a2[r][0].x;
        acc[r][1] = a2[r][0].y;
        acc[r][2] = a2[r][1].x;
        acc[r][3] = a2[r][1].y;
      }
#endif
      const float4 bb = *(const float4*)(b + 4 * jq);
      const float bs[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float v = __fadd_rn(acc[r][c], bs[c]);
          o[c] = relu ? (v < 0.0f ? 0.0f : v) : v;  // np.maximum(v, 0): NaN stays NaN
        }
        *(float4*)(y + (rq * 4 + r) * n_out + 4 * jq) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    return;
  }
  for (int t = threadIdx.x; t < rows * n_out; t += blockDim.x) {
    const int r = t / n_out, j = t - r * n_out;
    float acc = 0.0f;
#pragma unroll 8
    for (int k = 0; k < n_in; ++k) acc = fmaf(x[r * ldx + k], W[k * n_out + j], acc);
    const float v = __fadd_rn(acc, b[j]);
    y[r * n_out + j] = relu ? (v < 0.0f ? 0.0f : v) : v;
  }
}

__global__ void __launch_bounds__(kActThreads) actor_kernel(const __grid_constant__ ActorArgs a) {
  extern __shared__ __align__(16) float sa[];
  const int D0 = a.D0, H1 = a.H1, H2 = a.H2, A = a.A, L0 = a.L0, TR = a.rows;
  float* w1 = sa;                        // D0 x H1
  float* w2 = w1 + pad4(D0 * H1);        // H1 x H2
  float* w3 = w2 + pad4(H1 * H2);        // H2 x A
  float* b1 = w3 + pad4(H2 * A);
  float* b2 = b1 + pad4(H1);
  float* b3 = b2 + pad4(H2);
  float* xs = b3 + pad4(A);              // TR x L0 (then q: TR x A)
  float* h1 = xs + pad4(TR * L0 > TR * A ? TR * L0 : TR * A);  // TR x H1
  float* h2 = h1 + TR * H1;              // TR x H2
  uint64_t* bar = (uint64_t*)(h2 + TR * H2 + 4);
  float* qs = xs;
  const int nw[3] = {D0 * H1, H1 * H2, H2 * A};
  float* wd[3] = {w1, w2, w3};
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, 4u * (uint32_t)(nw[0] + nw[1] + nw[2]));
    for (int l = 0; l < 3; ++l) tma_bulk_g2s(wd[l], a.W[l], 4u * (uint32_t)nw[l], bar);
  }
  for (int j = threadIdx.x; j < H1; j += blockDim.x) b1[j] = a.b[0][j];
  for (int j = threadIdx.x; j < H2; j += blockDim.x) b2[j] = a.b[1][j];
  for (int j = threadIdx.x; j < A; j += blockDim.x) b3[j] = a.b[2][j];
  __syncthreads();
  mbar_wait(bar, 0);
  const int64_t tiles = (a.n + TR - 1) / TR;
  const int64_t vsize = vem_size(a.vem, a.t_step);
  // the next tile's states are loaded into registers while this tile
  // computes (kActPre per thread covers TR * L0 <= kActPre * blockDim)
  float pre[kActPre];
  auto load_tile = [&](int64_t tile) {
#pragma unroll
    for (int u = 0; u < kActPre; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      const int r = i / L0, k = i - r * L0;
      const int64_t row = tile * TR + r;
      pre[u] = (i < TR * L0 && k < D0 && row < a.n) ? a.states[row * D0 + k] : 0.0f;
    }
  };
  if (blockIdx.x < tiles) load_tile(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t row0 = tile * TR;
#pragma unroll
    for (int u = 0; u < kActPre; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      if (i < TR * L0) xs[i] = pre[u];
    }
    if (tile + gridDim.x < tiles) load_tile(tile + gridDim.x);  // lands during this tile
    __syncthreads();
    act_dense(xs, L0, D0, w1, b1, H1, h1, TR, true);
    __syncthreads();
    act_dense(h1, H1, H1, w2, b2, H2, h2, TR, true);
    __syncthreads();
    act_dense(h2, H2, H2, w3, b3, A, qs, TR, false);
    __syncthreads();
    for (int r = threadIdx.x; r < TR; r += blockDim.x) {
      const int64_t row = row0 + r;
      if (row >= a.n) continue;
      const float* q = qs + r * A;
      int best = 0;
      for (int j = 1; j < A; ++j)
        if (q[j] > q[best]) best = j;  // np.argmax: the first maximum
      const double eps = vem_epsilon_sized(a.vem, a.env0 + row, vsize);
      const double u = draw_uniform(stream_block(a.seed, a.lane, a.tag, a.ctr + (uint64_t)row),
                                    0.0, 1.0);
      const int64_t rnd = draw_integer(
          stream_block(a.seed, a.lane, a.tag, a.ctr + (uint64_t)a.n + (uint64_t)row), 0, A);
      a.actions[row] = u < eps ? rnd : (int64_t)best;
      if (a.q_out)
        for (int j = 0; j < A; ++j) a.q_out[row * A + j] = q[j];
    }
    __syncthreads();  // xs / qs are rewritten by the next tile
  }
}

__host__ __device__ __forceinline__ size_t actor_smem_bytes(int D0, int H1, int H2, int A,
                                                            int rows) {
  const int L0 = pad4(D0);
  const size_t fl = (size_t)pad4(D0 * H1) + pad4(H1 * H2) + pad4(H2 * A) + pad4(H1) + pad4(H2) +
                    pad4(A) + pad4(rows * L0 > rows * A ? rows * L0 : rows * A) +
                    (size_t)rows * H1 + (size_t)rows * H2 + 4;
  return fl * 4 + 16;
}

}  // namespace sp
