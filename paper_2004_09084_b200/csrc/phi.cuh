// phi.cuh -- the self-inverse check-node kernel Phi(x) = -ln tanh(x/2) on sm_100a.
//
// Reference: decoder.py:96-105 evaluates log1p(2/expm1(clip(x, eps, clip))) in FP64.
//
//  * phi_ref(double): the same formula on libdevice (the FP64 parity path).
//  * phi_fast(float): the FP32 hot-path version (see phi_fast_ge below).  Two libdevice
//    calls plus a division cost ~55 FP32 instructions per Phi and the update needs two
//    Phi per edge, which would make the kernel issue-bound far below the HBM roofline
//    (hard part 2).  With t = e^-x and d = 1 - t,
//        Phi(x) = ln((1 + t) / (1 - t)) = ln((2 - d) / d),
//    evaluated in three branch-free regions that keep ~1e-6 relative accuracy on the
//    whole range, including the tiny Phi values a degree-1-heavy check sums
//    (tests/test_device_parity.py::test_device_phi).  The long-run deviation of FP32
//    posteriors from the FP64 reference is dominated by FP32 rounding of the state
//    itself, not by this Phi.
#pragma once
#include <cuda_runtime.h>

namespace qcl {

__device__ __forceinline__ double phi_ref(double x, double eps, double clip) {
    x = fmin(fmax(x, eps), clip);
    return log1p(2.0 / expm1(x));
}

__device__ __forceinline__ float ex2_approx(float y) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
    return r;
}
__device__ __forceinline__ float lg2_approx(float y) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
    return r;
}
__device__ __forceinline__ float rcp_approx(float y) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
    return r;
}

// Phi for x >= eps (any upper value; callers clamp to the clip where the reference does).
//   region A, x < 1/16 : d = -expm1(-x) = x (1 - x/2 + x^2/6 - x^3/24 + x^4/120),
//                        truncation < 2e-9 relative; Phi = ln((2 - d) / d) via MUFU.LG2
//   region B, x < 2    : t = e^-x by MUFU.EX2, d = 1 - t (relative error <= 3e-6 at
//                        x = 1/16), Phi = ln((1 + t) / d)
//   region C, x >= 2   : Phi = 2 artanh(t) = t (2 + 2t^2/3 + 2t^4/5 + 2t^6/7 + 2t^8/9),
//                        t <= 0.136, truncation < 3e-10
// e^-x comes from ex2(x * -log2 e) without an exponent split: at the clip (x = 30) the
// rounding of the product costs 2.6e-6 relative on Phi ~ 1.9e-13, i.e. nothing once
// summed.  3 MUFU + ~20 FP32 instructions, branch free.
__device__ __forceinline__ float phi_fast_ge(float x) {
    const float kNegLog2e = -1.4426950408889634f;
    const float kLn2 = 0.6931471805599453f;
    float t = ex2_approx(x * kNegLog2e);
    float p = fmaf(x, 1.0f / 120.0f, -1.0f / 24.0f);
    p = fmaf(x, p, 1.0f / 6.0f);
    p = fmaf(x, p, -0.5f);
    p = fmaf(x, p, 1.0f);
    const float d = x < 0.0625f ? x * p : 1.0f - t;
    const float phi_log = lg2_approx((2.0f - d) * rcp_approx(d)) * kLn2;
    const float t2 = t * t;
    float s = fmaf(t2, 2.0f / 9.0f, 2.0f / 7.0f);
    s = fmaf(t2, s, 2.0f / 5.0f);
    s = fmaf(t2, s, 2.0f / 3.0f);
    s = fmaf(t2, s, 2.0f);
    return x >= 2.0f ? t * s : phi_log;
}

__device__ __forceinline__ float phi_fast(float x, float eps, float clip) {
    return phi_fast_ge(fminf(fmaxf(x, eps), clip));
}

// ---- lean pair used by the FP32 check update (two Phi per edge) -------------------
//
// Error model.  Outgoing messages r only need ABSOLUTE accuracy: r is added to q to
// form the posterior and subtracted next sweep, and every tolerance is relative to
// max(|ref|, 1).  A message error of ~1e-6 absolute is far inside the 1e-4 contract.
//
// phi_in(x) = Phi(x) / ln2 for x = |q| (log2 units).  ph_j only reaches the OTHER
//   edges' messages through Phi(others), whose slope is |Phi'(o)| = 1/sinh(o) <=
//   1/sinh(ph_j).  With d = 1 - t the absolute error of ph_j is ~1.7e-7 / x (t = e^-x
//   from MUFU.EX2), and 1/sinh(Phi(x)) ~ x for small x, so every message moves by
//   < 2e-7: no small-x branch is needed.  d is kept >= 0 (MUFU.EX2 may round e^-tiny
//   above 1); x = 0 gives ph = inf, which only drives the other messages' magnitudes
//   to 0 (reference: Phi(23.7 + ...) ~ 1e-10).  Large x (>= 4) uses the series
//   2t(1 + t^2/3), truncation < 3e-8 relative, because SMALL ph values are summed and
//   their relative accuracy matters.  12 instructions, 3 MUFU.
__device__ __forceinline__ float phi_in(float x) {
    const float kNegLog2e = -1.4426950408889634f;
    const float kInvLn2 = 1.4426950408889634f;
    const float t = ex2_approx(x * kNegLog2e);
    const float d = fmaxf(1.0f - t, 0.0f);
    const float lg = lg2_approx((1.0f + t) * rcp_approx(d));
    const float s = fmaf(t * t, 2.0f * kInvLn2 / 3.0f, 2.0f * kInvLn2);
    return x >= 4.0f ? t * s : lg;
}

// phi_out(y): Phi(x) in natural units for x = y ln2, y = others in log2 units, clamped
//   below at eps / ln2 by the caller (an upper clamp at the clip would change the
//   result by < Phi(clip) = 1.9e-13 and is omitted).  This is the outgoing magnitude:
//   x < 1/64 uses d = x (1 - x/2 + x^2/6) (truncation < 2e-7 relative, the large-message
//   regime), otherwise d = 1 - t (relative error <= 1.1e-5 at x = 1/64, i.e. <= 3e-6 on
//   Phi there).  For large x the logarithm of a ratio near 1 has ~2e-7 ABSOLUTE error,
//   which is all a message needs.  14 instructions, 3 MUFU.
__device__ __forceinline__ float phi_out(float y) {
    const float kLn2 = 0.6931471805599453f;
    const float t = ex2_approx(-y);
    // d = -expm1(-x) with x = y ln2: y (ln2 - ln2^2/2 y + ln2^3/6 y^2)
    const float p = fmaf(y, fmaf(y, 0.0555041086648216f, -0.2402265069591007f), kLn2);
    const float d = y < (1.0f / 64.0f) * 1.4426950408889634f ? y * p : 1.0f - t;
    return lg2_approx((2.0f - d) * rcp_approx(d)) * kLn2;
}

}  // namespace qcl
