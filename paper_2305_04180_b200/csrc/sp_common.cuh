// sp_common.cuh -- shared device code for the Sparrow B200 kernels.
//
// * Philox4x32-10 counter-based streams and the draw mappings of the RNG
//   contract, which stand in for the reference's
//   per-lane numpy streams (vecenv.py:86-89, params.py:112-121, core.py:136-138,
//   core.py:240, replay.py:76).
// * Exact-rounding fp64 helpers: the env math is written with __d*_rn
//   intrinsics so no FMA contraction changes the reference's rounding
//   (numpy evaluates k*v + (1-k)*m etc. with separate roundings).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

#include "../../include/sparrow.h"

#define SP_PI 3.141592653589793
#define SP_TWO_PI 6.283185307179586
#define SP_INV_PI 0.3183098861837907  // 1 / SP_PI, correctly rounded
#define SP_FULL 0xffffffffu

// SP_CHECKED builds (tools/gpu_checked.sh): device-side bounds checks on
// the step kernel's shared-memory slots, queue entries, table cells and
// output rows -- compute-sanitizer is closed on this pool, so the checks
// are our own.  A failed check prints its site and traps.
#ifdef SP_CHECKED
#include <cstdio>
#define SP_CHECK(cond)                                                              \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("SP_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                          \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define SP_CHECK(cond) \
  do {             \
  } while (0)
#endif

namespace sp {

// ---------------------------------------------------------------- Philox ---
struct Block4 {
  uint32_t x0, x1, x2, x3;
};

__device__ __forceinline__ Block4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Block4{c0, c1, c2, c3};
}

// One stream = (seed, lane, tag); `ctr` counts blocks.
__device__ __forceinline__ Block4 stream_block(uint64_t seed, uint32_t lane, uint32_t tag,
                                               uint64_t ctr) {
  return philox4x32_10((uint32_t)ctr, (uint32_t)(ctr >> 32), lane, tag, (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

__device__ __forceinline__ uint64_t word64(const Block4& b) {
  return ((uint64_t)b.x1 << 32) | b.x0;
}

// numpy Generator.uniform arithmetic: lo + (hi - lo) * u53
__device__ __forceinline__ double draw_uniform(const Block4& b, double lo, double hi) {
  double u = (double)(word64(b) >> 11) * 0x1.0p-53;
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

// integers(lo, hi), hi exclusive: lo + mulhi64(w, hi - lo)
__device__ __forceinline__ int64_t draw_integer(const Block4& b, int64_t lo, int64_t hi) {
  return lo + (int64_t)__umul64hi(word64(b), (uint64_t)(hi - lo));
}

// -2 ln(u1), u1 = (x + 1) / 2^32 in (0, 1], to fp32 relative precision: for
// u1 >= 1/2 through log1p of the exact integer complement (a plain fp32 u1
// would keep only 24 of the 32 bits and lose r = sqrt(-2 ln u1) near u1 = 1).
__device__ __forceinline__ float neg2log_u1(uint32_t x) {
  if (x >= 0x80000000u) return -2.0f * log1pf(-(float)(0xFFFFFFFFu - x) * 0x1.0p-32f);
  return -2.0f * logf(((float)x + 1.0f) * 0x1.0p-32f);
}

// Four standard normals per block (Box-Muller on (x0,x1), (x2,x3)), the RNG
// contract's mapping (oracle or_normals) evaluated in fp32: z is within
// ~5e-7 absolute of the fp64 value (|z| <= 6.7), i.e. a noisy range within
// sigma * 5e-7 cm.  The noise never feeds a branch.
__device__ __forceinline__ void draw_normals4(const Block4& b, float z[4]) {
  float ra = sqrtf(neg2log_u1(b.x0));
  float rb = sqrtf(neg2log_u1(b.x2));
  float sa, ca, sb, cb;
  sincospif(2.0f * ((float)b.x1 * 0x1.0p-32f), &sa, &ca);
  sincospif(2.0f * ((float)b.x3 * 0x1.0p-32f), &sb, &cb);
  z[0] = ra * ca;
  z[1] = ra * sa;
  z[2] = rb * cb;
  z[3] = rb * sb;
}

// ----------------------------------------------------------- fp64 helpers ---
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dclip(double v, double lo, double hi) {
  return fmin(fmax(v, lo), hi);
}

// kinematics.py:17-19: pi - np.mod(pi - a, 2 pi)   (np.mod = fmod + sign fix).
// For |pi - a| < 4 pi (every heading update) fmod's exact remainder is b or
// b - 2 pi, and b - 2 pi is exact there (Sterbenz), so the fast path gives the
// same bits without the fmod loop; anything else takes the general path.
__device__ __forceinline__ double wrap_angle(double a) {
  const double b = dsub(SP_PI, a);
  if (b > -SP_TWO_PI && b < 2.0 * SP_TWO_PI) {
    if (b == 0.0) return SP_PI;                                  // m = +0
    if (b < 0.0) return dsub(SP_PI, dadd(b, SP_TWO_PI));         // sign fix
    return dsub(SP_PI, b < SP_TWO_PI ? b : dsub(b, SP_TWO_PI));  // fmod, exact
  }
  double m = fmod(b, SP_TWO_PI);
  if (m != 0.0) {
    if (m < 0.0) m = dadd(m, SP_TWO_PI);
  } else {
    m = 0.0;
  }
  return dsub(SP_PI, m);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace sp
