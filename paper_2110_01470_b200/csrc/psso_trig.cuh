// psso_trig.cuh -- branch-free trig for the register-resident chain kernel.
//
// The objectives' transcendental terms (benchmarks.py:128-140 cos(2*pi*x),
// :165-166 sin(sqrt|x|)) dominate the issue budget of the fused iteration
// once the keyed hash is paid for.  These versions use an exact argument
// reduction and one near-minimax polynomial (coefficients from
// scripts/fit_trig.py, max abs error 1.4e-16 / 3.8e-17 in fp64 before
// rounding of the Horner steps), no range branch and no libdevice call:
//
//   cos(2*pi*x):  s = 2x - rint(2x) exactly (|s| <= 1/2),
//                 cos(2*pi*x) = (-1)^rint(2x) * P(s^2)        -- 12 fp64 ops
//   sin(w):       r = w - k*pi (two-constant Cody-Waite, FMA), |r| <= pi/2,
//                 sin(w) = (-1)^k * r * Q(r^2)                 -- 15 fp64 ops
//
// Validity: |2x| < 2^51 (cos) and |w| < 2^40 (sin).  The chain kernel only
// evaluates positions inside the search box, and psso_create selects it only
// when the box satisfies these bounds (otherwise the tile kernels, whose
// fast_cos/fast_sin fall back to libdevice, run).  Agreement with numpy's
// cos(fl(2*pi*x)) is to a few 1e-15 absolute per term, far inside the
// 1e-12 relative fitness tolerance of the transcendental objectives.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace psso {

// cos(pi*s) = P(s^2), |s| <= 1/2
static __constant__ double kCosPiD[9] = {
    1.0, -4.934802200544676, 4.058712126416498, -1.335262768843456, 0.23533063012967062,
    -0.02580688873817758, 0.001929556278037417, -0.00010456656706174584, 4.149578027057121e-06};
static __constant__ float kCosPiF[6] = {1.0f, -4.934802055358887f, 4.058709144592285f,
                                        -1.335211992263794f, 0.23493731021881104f,
                                        -0.024396324530243874f};
// sin(r) = r * Q(r^2), |r| <= pi/2
static __constant__ double kSinQD[10] = {
    1.0, -0.16666666666666666, 0.008333333333333333, -0.0001984126984126967,
    2.7557319223940737e-06, -2.5052108378604874e-08, 1.6059043206485008e-10,
    -7.647127747343607e-13, 2.810214694451185e-15, -7.982533321458908e-18};
static __constant__ float kSinQF[6] = {1.0f, -0.1666666716337204f, 0.008333330973982811f,
                                       -0.00019840861205011606f, 2.752528644123231e-06f,
                                       -2.3889498379503493e-08f};

template <typename T> struct Trig;

template <> struct Trig<double> {
  // |cos(2*pi*x)| polynomial value and the parity bit of rint(2x) (sign = -1 if odd)
  static __device__ __forceinline__ double cos2pi_abs(double x, uint32_t& odd) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __fma_rn(x, 2.0, M);
    const double kd = __dsub_rn(t, M);
    odd = (uint32_t)__double2loint(t) << 31;
    const double s = __fma_rn(x, 2.0, -kd);  // exact
    const double z = __dmul_rn(s, s);
    double p = kCosPiD[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) p = __fma_rn(p, z, kCosPiD[i]);
    return p;
  }
  static __device__ __forceinline__ double flip(double v, uint32_t odd) {
    return __hiloint2double(__double2hiint(v) ^ (int)odd, __double2loint(v));
  }
  static __device__ __forceinline__ double cos2pi(double x) {
    uint32_t odd;
    const double p = cos2pi_abs(x, odd);
    return flip(p, odd);
  }
  // cos(y), |y| < 2^40: k = rint(y/pi), r = y - k*pi (two-constant Cody-Waite),
  // cos(y) = (-1)^k cos(pi * s) with s = r/pi, |s| <= 1/2 -- the cos(pi s)
  // polynomial again (f7's cos(x_j / sqrt(j)))
  static __device__ __forceinline__ double cos_(double y) {
    const double M = 6755399441055744.0;
    const double t = __fma_rn(y, 0.3183098861837907, M);  // 1/pi
    const double kd = __dsub_rn(t, M);
    const uint32_t odd = (uint32_t)__double2loint(t) << 31;
    double r = __fma_rn(-kd, 3.141592653589793, y);
    r = __fma_rn(-kd, 1.2246467991473532e-16, r);
    const double sp = __dmul_rn(r, 0.3183098861837907);
    const double z = __dmul_rn(sp, sp);
    double p = kCosPiD[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) p = __fma_rn(p, z, kCosPiD[i]);
    return flip(p, odd);
  }
  static __device__ __forceinline__ double sin_(double w) {
    const double M = 6755399441055744.0;
    const double t = __fma_rn(w, 0.3183098861837907, M);  // 1/pi
    const double kd = __dsub_rn(t, M);
    const uint32_t odd = (uint32_t)__double2loint(t) << 31;
    double r = __fma_rn(-kd, 3.141592653589793, w);
    r = __fma_rn(-kd, 1.2246467991473532e-16, r);
    const double z = __dmul_rn(r, r);
    double q = kSinQD[9];
#pragma unroll
    for (int i = 8; i >= 0; --i) q = __fma_rn(q, z, kSinQD[i]);
    return flip(__dmul_rn(r, q), odd);
  }
};

template <> struct Trig<float> {
  static __device__ __forceinline__ float cos2pi_abs(float x, uint32_t& odd) {
    const float M = 12582912.0f;  // 1.5 * 2^23
    const float t = __fmaf_rn(x, 2.0f, M);
    const float kd = __fsub_rn(t, M);
    odd = (uint32_t)__float_as_uint(t) << 31;
    const float s = __fmaf_rn(x, 2.0f, -kd);
    const float z = __fmul_rn(s, s);
    float p = kCosPiF[5];
#pragma unroll
    for (int i = 4; i >= 0; --i) p = __fmaf_rn(p, z, kCosPiF[i]);
    return p;
  }
  static __device__ __forceinline__ float flip(float v, uint32_t odd) {
    return __uint_as_float(__float_as_uint(v) ^ odd);
  }
  static __device__ __forceinline__ float cos2pi(float x) {
    uint32_t odd;
    const float p = cos2pi_abs(x, odd);
    return flip(p, odd);
  }
  static __device__ __forceinline__ float cos_(float y) {
    const float M = 12582912.0f;
    const float t = __fmaf_rn(y, 0.31830987334251404f, M);
    const float kd = __fsub_rn(t, M);
    const uint32_t odd = (uint32_t)__float_as_uint(t) << 31;
    float r = __fmaf_rn(-kd, 3.1415927410125732f, y);
    r = __fmaf_rn(-kd, -8.742277657347586e-08f, r);
    const float sp = __fmul_rn(r, 0.31830987334251404f);
    const float z = __fmul_rn(sp, sp);
    float p = kCosPiF[5];
#pragma unroll
    for (int i = 4; i >= 0; --i) p = __fmaf_rn(p, z, kCosPiF[i]);
    return flip(p, odd);
  }
  static __device__ __forceinline__ float sin_(float w) {
    const float M = 12582912.0f;
    const float t = __fmaf_rn(w, 0.31830987334251404f, M);
    const float kd = __fsub_rn(t, M);
    const uint32_t odd = (uint32_t)__float_as_uint(t) << 31;
    float r = __fmaf_rn(-kd, 3.1415927410125732f, w);
    r = __fmaf_rn(-kd, -8.742277657347586e-08f, r);
    const float z = __fmul_rn(r, r);
    float q = kSinQF[5];
#pragma unroll
    for (int i = 4; i >= 0; --i) q = __fmaf_rn(q, z, kSinQF[i]);
    return flip(__fmul_rn(r, q), odd);
  }
};

// Largest |position| for which the chain kernel's trig is valid (host check).
constexpr double kChainTrigMaxAbs = 1.0e12;
constexpr double kChainTrigMaxAbsF32 = 1.0e6;  // fp32: |2x| < 2^22, Cody-Waite in fp32

}  // namespace psso
