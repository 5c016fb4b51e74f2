// sp_learn.cu -- one double-DQN update of the [D0, H1, H2, A] ReLU MLP in three
// launches (the reference's ddqn.py:38-77 + net.py:63-161).
//
//   ddqn_rows_kernel   row-parallel, one CTA per TR-row tile of the batch.  The
//                      weights are staged per layer into shared memory by TMA
//                      bulk copies, triple-buffered (W1 | W2 | W3), then:
//                        targets  y = r + gamma (1-d) Q_tgt(s', argmax Q_on(s'))
//                        forward  Q_on(s) keeping activations
//                        Huber(1) gradient dq on q[i, a_i] (mean over B)
//                        deltas   d2 = (dq W3^T)[z2>0], d1 = (d2 W2^T)[z1>0]
//                      a1, a2, dq, d2, d1 go to a global scratch (B rows each).
//   ddqn_grad_adam_kernel  the weight gradients as 32x64 GEMM tiles over the
//                      batch (rows in order: deterministic), Adam fused into the
//                      epilogue (adam_kernel's gated update).
//   adam_tick_stats_kernel   advances the device Adam step when the loss is finite.
//
// Everything is fp32, the reference's numpy dtype, with its elementwise
// operation order.  ReLU propagates NaN as np.maximum does, so a diverged
// batch reaches the finite-loss gate (ddqn.py:66-71).  Matmul sums run in a
// fixed order (k ascending), which differs from BLAS blocking in the last bits
// only.  The tests hold this path to the torch path's bar: 1e-4 after 12
// updates.  Parameters are the Adam tensor order of asl._adam_launch:
// W1 W2 W3 b1 b2 b3.
#pragma once
#include "sp_common.cuh"

namespace sp {

constexpr int kLearnThreads = 256;
constexpr int kLearnMaxD0 = 128, kLearnMaxH = 256, kLearnMaxA = 16;

struct MlpDev {
  const float* W[3];  // (D0,H1) (H1,H2) (H2,A) row-major, as net.py stores them
  const float* b[3];
};

struct LearnArgs {
  MlpDev on, tgt;
  const float* s;       // (B, D0)
  const int64_t* a;     // (B,)
  const float* r;       // (B,)
  const float* s2;      // (B, D0)
  const uint8_t* d;     // (B,)
  float *a1, *a2, *dq, *d1, *d2;  // (B,H1) (B,H2) (B,A) (B,H1) (B,H2) scratch
  float* lpart;         // (n_tiles, 2): sum of Huber terms, sum of |td|
  int B, D0, H1, H2, A;
  float gamma;
};

__device__ __forceinline__ float relu_nan(float v) { return v < 0.0f ? 0.0f : v; }

__host__ __device__ __forceinline__ int pad4(int n) { return (n + 3) & ~3; }

// Weight staging, triple-buffered: one shared-memory buffer (and mbarrier)
// per layer, each filled by a single TMA bulk copy (cp.async.bulk, issued by
// thread 0).  Because each layer always uses its own buffer, the next pass's
// layer-l weights stream in as soon as this pass's layer l is done, behind
// the other layers' math.  The online net's W2/W3 stay resident after the
// last pass for the backward.  W1's buffer holds pad4(D0) rows; the pad rows
// are zeroed once and never written by the copies.
struct Stager {
  float* buf[3];
  uint64_t* bar[3];
  uint32_t phase[3];

  // thread 0 only; the buffer's previous readers must have passed a barrier
  __device__ __forceinline__ void issue(int l, const float* src, int n_floats) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar[l], (uint32_t)n_floats * 4u);
    tma_bulk_g2s(buf[l], src, (uint32_t)n_floats * 4u, bar[l]);
  }
  // every thread
  __device__ __forceinline__ void wait(int l) {
    mbar_wait(bar[l], phase[l]);
    phase[l] ^= 1u;
  }
};

template <int TR>
__host__ __device__ __forceinline__ int learn_part_floats(int L0, int H1, int H2) {
  // split-K partials of a dense layer: splits * TR * n_out <= 4 * threads * TR
  (void)L0; (void)H1; (void)H2;
  return 4 * kLearnThreads * TR;
}

// y[r][j] = b[j] + sum_k x[r][k] Ws[k][j] (Ws staged in SMEM) for the TR rows.
// n_out % 4 == 0: thread = (4-column quad, k-split).  Each thread reads each of
// its weights once (float4) and applies it to all TR rows (x rows read as
// float4, broadcast across the warp), so shared-memory traffic is one weight
// word per TR FMAs.  The k-split partials meet in `part` and are summed in
// split order (deterministic).  n_in is the padded row stride of x (% 4 == 0).
// Otherwise (the A-wide output layer) one thread per (row, column).
template <int TR>
__device__ __forceinline__ void dense_smem(const float* Ws, const float* __restrict__ bias,
                                           const float* x, int n_in, int n_out, float* y, float* z,
                                           bool relu, float* part) {
  if ((n_out & 3) == 0) {
    const int quads = n_out >> 2;
    const int splits = max(1, min((int)blockDim.x / quads, n_in >> 2));
    const int kq = ((n_in >> 2) + splits - 1) / splits;  // k-quads per split
    for (int t = threadIdx.x; t < quads * splits; t += blockDim.x) {
      const int jq = t % quads, sp = t / quads;
      const int kb = 4 * sp * kq, ke = min(n_in, kb + 4 * kq);
      float acc[TR][4];
#pragma unroll
      for (int q = 0; q < TR; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[q][c] = 0.0f;
      for (int k = kb; k < ke; k += 4) {
        float4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = *(const float4*)(Ws + (k + u) * n_out + 4 * jq);
#pragma unroll
        for (int q = 0; q < TR; ++q) {
          const float4 xv = *(const float4*)(x + q * n_in + k);
          const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc[q][0] = fmaf(xs[u], w[u].x, acc[q][0]);
            acc[q][1] = fmaf(xs[u], w[u].y, acc[q][1]);
            acc[q][2] = fmaf(xs[u], w[u].z, acc[q][2]);
            acc[q][3] = fmaf(xs[u], w[u].w, acc[q][3]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < TR; ++q)
        *(float4*)(part + (sp * TR + q) * n_out + 4 * jq) =
            make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
    }
    __syncthreads();
    const int stride = TR * n_out;
    for (int e = threadIdx.x; e < stride; e += blockDim.x) {
      const int j = (n_out & (n_out - 1)) == 0 ? (e & (n_out - 1)) : e % n_out;
      float v = part[e];
      for (int sp = 1; sp < splits; ++sp) v += part[sp * stride + e];
      v += bias[j];  // x @ W + b (net.py:63-74)
      if (z) z[e] = v;
      y[e] = relu ? relu_nan(v) : v;
    }
    return;
  }
  for (int t = threadIdx.x; t < TR * n_out; t += blockDim.x) {
    const int r = t / n_out, jj = t - r * n_out;
    float acc = 0.0f;
    for (int k = 0; k < n_in; ++k) acc = fmaf(x[r * n_in + k], Ws[k * n_out + jj], acc);
    const float v = acc + bias[jj];
    if (z) z[r * n_out + jj] = v;
    y[r * n_out + jj] = relu ? relu_nan(v) : v;
  }
}

// One forward pass over the TR rows.  `next` (nullable): the net of the next
// pass, whose layer-l weights are issued into buffer l right after this pass
// has finished layer l.
template <int TR>
__device__ __forceinline__ void mlp_forward(const MlpDev& m, const MlpDev* next, const float* x,
                                            float* h1, float* h2, float* q, float* z1, float* z2,
                                            Stager& st, float* part, const LearnArgs& a) {
  const int n[3] = {a.D0 * a.H1, a.H1 * a.H2, a.H2 * a.A};
  st.wait(0);
  dense_smem<TR>(st.buf[0], m.b[0], x, pad4(a.D0), a.H1, h1, z1, true, part);
  __syncthreads();
  if (next && threadIdx.x == 0) st.issue(0, next->W[0], n[0]);
  st.wait(1);
  dense_smem<TR>(st.buf[1], m.b[1], h1, a.H1, a.H2, h2, z2, true, part);
  __syncthreads();
  if (next && threadIdx.x == 0) st.issue(1, next->W[1], n[1]);
  st.wait(2);
  dense_smem<TR>(st.buf[2], m.b[2], h2, a.H2, a.A, q, nullptr, false, part);
  __syncthreads();
  if (next && threadIdx.x == 0) st.issue(2, next->W[2], n[2]);
}

template <int TR>
__global__ void __launch_bounds__(kLearnThreads)
    ddqn_rows_kernel(const __grid_constant__ LearnArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int D0 = a.D0, H1 = a.H1, H2 = a.H2, A = a.A, L0 = pad4(D0);
  Stager st;
  st.buf[0] = sm;                                  // W1: pad4(D0) x H1
  st.buf[1] = st.buf[0] + pad4(L0 * H1);           // W2: H1 x H2
  st.buf[2] = st.buf[1] + pad4(H1 * H2);           // W3: H2 x A
  float* part = st.buf[2] + pad4(H2 * A);          // split-K partials (learn_part_floats)
  float* xs = part + learn_part_floats<TR>(L0, H1, H2);  // TR x L0  s rows (zero-padded)
  float* xs2 = xs + TR * L0;                 // TR x L0   s' rows
  float* h1 = xs2 + TR * L0;                 // TR x H1
  float* h2 = h1 + TR * H1;                  // TR x H2
  float* z1 = h2 + TR * H2;                  // TR x H1   online(s) pre-activations
  float* z2 = z1 + TR * H1;                  // TR x H2
  float* q = z2 + TR * H2;                   // TR x A
  float* dq = q + TR * A;                    // TR x A
  float* d2 = dq + TR * A;                   // TR x H2
  float* y = d2 + TR * H2;                   // TR
  float* red = y + TR;                       // 2 x TR
  uint64_t* bars = (uint64_t*)(sm + pad4((int)(red + 2 * TR - sm)));  // 16-byte aligned
  for (int l = 0; l < 3; ++l) {
    st.bar[l] = bars + l;
    st.phase[l] = 0;
  }
  for (int i = D0 * H1 + threadIdx.x; i < L0 * H1; i += blockDim.x) st.buf[0][i] = 0.0f;
  if (threadIdx.x == 0) {
    for (int l = 0; l < 3; ++l) mbar_init(st.bar[l], 1);
    st.issue(0, a.on.W[0], D0 * H1);  // the first pass's weights
    st.issue(1, a.on.W[1], H1 * H2);
    st.issue(2, a.on.W[2], H2 * A);
  }
  const int row0 = blockIdx.x * TR;
  for (int i = threadIdx.x; i < TR * L0; i += blockDim.x) {
    const int r = i / L0, k = i - r * L0;
    xs[i] = k < D0 ? a.s[(size_t)(row0 + r) * D0 + k] : 0.0f;
    xs2[i] = k < D0 ? a.s2[(size_t)(row0 + r) * D0 + k] : 0.0f;
  }
  __syncthreads();
  // ---- targets (ddqn.py:38-51): argmax of the online net, value of the target net
  mlp_forward<TR>(a.on, &a.tgt, xs2, h1, h2, q, nullptr, nullptr, st, part, a);
  if (threadIdx.x < TR) {
    const int r = threadIdx.x;
    int best = 0;
    for (int j = 1; j < A; ++j)
      if (q[r * A + j] > q[r * A + best]) best = j;  // first max, as np.argmax
    y[r] = (float)best;
  }
  __syncthreads();
  mlp_forward<TR>(a.tgt, &a.on, xs2, h1, h2, q, nullptr, nullptr, st, part, a);
  if (threadIdx.x < TR) {
    const int r = threadIdx.x;
    const float boot = q[r * A + (int)y[r]];
    const float nd = a.d[row0 + r] ? 0.0f : 1.0f;
    y[r] = __fadd_rn(a.r[row0 + r], __fmul_rn(__fmul_rn(a.gamma, nd), boot));
  }
  __syncthreads();
  // ---- online forward on s, cached (net.py:63-74); W3 stays staged below
  mlp_forward<TR>(a.on, nullptr, xs, h1, h2, q, z1, z2, st, part, a);
  // ---- Huber(1) on q[r, a_r] - y_r (net.py:83-115): mean over the batch
  if (threadIdx.x < TR) {
    const int r = threadIdx.x;
    const int act = (int)a.a[row0 + r];
    const float res = __fsub_rn(q[r * A + act], y[r]);
    const float ab = fabsf(res);
    red[r] = ab <= 1.0f ? __fmul_rn(__fmul_rn(0.5f, res), res) : __fsub_rn(ab, 0.5f);
    red[TR + r] = ab;
    const float g = __fdiv_rn(fminf(fmaxf(res, -1.0f), 1.0f), (float)a.B);
    for (int j = 0; j < A; ++j) dq[r * A + j] = j == act ? g : 0.0f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float l = 0.0f, m = 0.0f;
    for (int r = 0; r < TR; ++r) {
      l += red[r];
      m += red[TR + r];
    }
    a.lpart[blockIdx.x * 2] = l;
    a.lpart[blockIdx.x * 2 + 1] = m;
  }
  // activations and dq for the parameter-parallel gradient kernel
  for (int i = threadIdx.x; i < TR * H1; i += blockDim.x) a.a1[(size_t)row0 * H1 + i] = h1[i];
  for (int i = threadIdx.x; i < TR * H2; i += blockDim.x) a.a2[(size_t)row0 * H2 + i] = h2[i];
  for (int i = threadIdx.x; i < TR * A; i += blockDim.x) a.dq[(size_t)row0 * A + i] = dq[i];
  // ---- d2 = (dq W3^T) * [z2 > 0]   (the online W3 is still staged)
  const float* wbuf = st.buf[2];
  for (int e = threadIdx.x; e < TR * H2; e += blockDim.x) {
    const int r = e / H2, k = e - r * H2;
    float acc = 0.0f;
    for (int j = 0; j < A; ++j) acc = fmaf(dq[r * A + j], wbuf[k * A + j], acc);
    const float v = z2[e] > 0.0f ? acc : 0.0f;
    d2[e] = v;
    a.d2[(size_t)row0 * H2 + e] = v;
  }
  __syncthreads();
  // ---- d1 = (d2 W2^T) * [z1 > 0] with the online W2 still staged; thread k
  // walks row k starting at column k (rotated), so a warp's 32 rows hit 32
  // different banks
  __syncthreads();
  const float* w2s = st.buf[1];
  for (int k = threadIdx.x; k < H1; k += blockDim.x) {
    float acc[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) acc[r] = 0.0f;
    const float* wrow = w2s + k * H2;
    int j = k % H2;
    for (int jj = 0; jj < H2; ++jj) {
      const float w = wrow[j];
#pragma unroll
      for (int r = 0; r < TR; ++r) acc[r] = fmaf(d2[r * H2 + j], w, acc[r]);
      j = j + 1 == H2 ? 0 : j + 1;
    }
#pragma unroll
    for (int r = 0; r < TR; ++r)
      a.d1[(size_t)(row0 + r) * H1 + k] = z1[r * H1 + k] > 0.0f ? acc[r] : 0.0f;
  }
}

// Weight gradients as small GEMMs over the batch, Adam fused into the epilogue.
// A CTA owns a 16 (fan_in) x 16 (fan_out) tile of one weight matrix:
//   gW[k][j] = sum_r act[r][k] del[r][j]   (W1: s, d1; W2: a1, d2; W3: a2, dq)
// with the tile's columns of all B rows staged in shared memory (B x 32 floats);
// each thread owns one output.  Tiles at k0 == 0 also own the bias gradient sum_r del[r][j].
// The sums run in row order (deterministic).  Then adam_kernel's update
// (net.py:141-161), gated on a finite loss (ddqn.py:66-71).  CTA 0 publishes
// {loss, mean |td|}.
constexpr int kGradTK = 16, kGradTJ = 16, kMaxGradTiles = 512;

struct GradTiles {
  int n;
  uint8_t tensor[kMaxGradTiles];  // 0..2: W1 W2 W3
  int16_t k0[kMaxGradTiles], j0[kMaxGradTiles];
};

__device__ __forceinline__ void adam_one(const AdamTensors& T, int k, int64_t e, float g,
                                         float c1, float c2, float fb1, float fb2, float f1b1,
                                         float f1b2, float flr, float feps) {
  const float mm = __fadd_rn(__fmul_rn(T.m[k][e], fb1), __fmul_rn(f1b1, g));
  const float vv = __fadd_rn(__fmul_rn(T.v[k][e], fb2), __fmul_rn(f1b2, __fmul_rn(g, g)));
  T.m[k][e] = mm;
  T.v[k][e] = vv;
  const float upd = __fdiv_rn(__fmul_rn(flr, __fdiv_rn(mm, c1)),
                              __fadd_rn(__fsqrt_rn(__fdiv_rn(vv, c2)), feps));
  T.p[k][e] = __fsub_rn(T.p[k][e], upd);
}

__global__ void __launch_bounds__(256)
    ddqn_grad_adam_kernel(const __grid_constant__ LearnArgs la,
                          const __grid_constant__ AdamTensors T,
                          const __grid_constant__ GradTiles tiles, int n_row_tiles,
                          const double* step_dev, double lr, double b1, double b2, double eps,
                          float* stats_out) {
  extern __shared__ __align__(16) float gsm[];  // As: B x kGradTK, Ds: B x kGradTJ
  __shared__ float stat_s[2];
  if (threadIdx.x < 32) {  // the row tiles' loss partials: lane-strided sums + xor tree
    float l = 0.0f, m = 0.0f;
    for (int t = threadIdx.x; t < n_row_tiles; t += 32) {
      l += la.lpart[2 * t];
      m += la.lpart[2 * t + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l += __shfl_xor_sync(SP_FULL, l, o);
      m += __shfl_xor_sync(SP_FULL, m, o);
    }
    if (threadIdx.x == 0) {
      stat_s[0] = l / (float)la.B;
      stat_s[1] = m / (float)la.B;
    }
  }
  __syncthreads();
  const float loss = stat_s[0], mad = stat_s[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    stats_out[0] = loss;
    stats_out[1] = mad;
  }
  if (!isfinite(loss)) return;  // uniform across the grid
  const int tk = tiles.tensor[blockIdx.x], k0 = tiles.k0[blockIdx.x], j0 = tiles.j0[blockIdx.x];
  const float* act = tk == 0 ? la.s : tk == 1 ? la.a1 : la.a2;
  const float* del = tk == 0 ? la.d1 : tk == 1 ? la.d2 : la.dq;
  const int K = tk == 0 ? la.D0 : tk == 1 ? la.H1 : la.H2;
  const int J = tk == 0 ? la.H1 : tk == 1 ? la.H2 : la.A;
  const int kk = threadIdx.x >> 4, jp = threadIdx.x & 15;  // output (k0+kk, j0+jp)
  float acc = 0.f, bacc = 0.f;
  const bool bias_owner = k0 == 0 && kk == 0;
  // the tile's columns of every batch row, staged once (many loads in flight)
  float* As = gsm;
  float* Ds = gsm + (size_t)la.B * kGradTK;
  for (int i = threadIdx.x; i < la.B * kGradTK; i += blockDim.x) {
    const int r = i / kGradTK, c = i % kGradTK;
    As[i] = k0 + c < K ? act[(size_t)r * K + k0 + c] : 0.0f;
  }
  if ((J & 3) == 0 && (j0 & 3) == 0) {
    for (int i = threadIdx.x; i < la.B * (kGradTJ / 4); i += blockDim.x) {
      const int r = i / (kGradTJ / 4), c = 4 * (i % (kGradTJ / 4));
      *(float4*)&Ds[r * kGradTJ + c] = j0 + c < J ? *(const float4*)&del[(size_t)r * J + j0 + c]
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    for (int i = threadIdx.x; i < la.B * kGradTJ; i += blockDim.x) {
      const int r = i / kGradTJ, c = i % kGradTJ;
      Ds[i] = j0 + c < J ? del[(size_t)r * J + j0 + c] : 0.0f;
    }
  }
  __syncthreads();
#pragma unroll 8
  for (int r = 0; r < la.B; ++r) {
    const float dv = Ds[r * kGradTJ + jp];
    acc = fmaf(As[r * kGradTK + kk], dv, acc);
    if (bias_owner) bacc += dv;
  }
  const double t = *step_dev + 1.0;
  const float c1 = (float)(1.0 - pow(b1, t));
  const float c2 = (float)(1.0 - pow(b2, t));
  const float fb1 = (float)b1, fb2 = (float)b2, f1b1 = (float)(1.0 - b1),
              f1b2 = (float)(1.0 - b2), flr = (float)lr, feps = (float)eps;
  const int k = k0 + kk, j = j0 + jp;
  if (k < K && j < J) adam_one(T, tk, (int64_t)k * J + j, acc, c1, c2, fb1, fb2, f1b1, f1b2, flr, feps);
  if (bias_owner && j < J) adam_one(T, tk + 3, j, bacc, c1, c2, fb1, fb2, f1b1, f1b2, flr, feps);
}

__global__ void adam_tick_stats_kernel(double* step_dev, const float* stats) {
  if (isfinite(stats[0])) *step_dev += 1.0;
}

template <int TR>
size_t learn_smem_bytes(int D0, int H1, int H2, int A) {
  const int L0 = pad4(D0);
  const size_t floats = (size_t)pad4(L0 * H1) + pad4(H1 * H2) + pad4(H2 * A) +
                        learn_part_floats<TR>(L0, H1, H2) +
                        (size_t)TR * (2 * L0 + 2 * H1 + 3 * H2 + 2 * A + 1) + 2 * TR;
  return sizeof(float) * (size_t)pad4((int)floats) + 3 * 8 + 16;
}

}  // namespace sp
