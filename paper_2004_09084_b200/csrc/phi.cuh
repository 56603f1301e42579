// phi.cuh -- the self-inverse check-node kernel Phi(x) = -ln tanh(x/2) on sm_100a.
//
// Reference: decoder.py:96-105 evaluates log1p(2/expm1(clip(x, eps, clip))) in FP64.
//
//  * phi_ref(double): the same formula on libdevice (the FP64 parity path).
//  * phi_fast(float): the FP32 hot-path version.  Two libdevice calls plus a
//    division cost ~55 FP32 instructions per Phi and the update needs two Phi per
//    edge, which would make the kernel issue-bound below the HBM roofline
//    (hard part 2).  Instead, with t = e^-x and d = 1 - t:
//
//        Phi(x) = ln((1 + t) / (1 - t)) = ln((2 - d) / d)
//
//      region A, x < 0.25 : d = -expm1(-x) by its Taylor series (degree 7,
//                           truncation < 5e-8 relative), ln via MUFU.LG2 of an
//                           argument >= 8, so the log has full relative accuracy;
//      region B, x < 2    : t from MUFU.EX2, d = 1 - t (t <= 0.78, no cancellation),
//                           ln via MUFU.LG2 of (1+t)/d in [1.31, 8.1];
//      region C, x >= 2   : Phi = 2 artanh(t) = 2t(1 + t^2/3 + t^4/5 + t^6/7 + t^8/9)
//                           (t <= 0.136, truncation < 3e-10), which keeps relative
//                           accuracy on the tiny Phi values a degree-1 check sums.
//    The exponent x*log2(e) is formed as hi + lo with an FMA so e^-x keeps ~1e-7
//    relative accuracy up to the clip (30).  Max relative error over [eps, clip]
//    is ~5e-7 for fp32 inputs (tests/test_device_parity.py::test_device_phi_fp32); the long-run
//    deviation of FP32 posteriors from the FP64 reference is dominated by
//    FP32 rounding of the state itself, not by this Phi.
//    Branch-free: 3 MUFU + ~23 FP32 ops.
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

__device__ __forceinline__ float phi_fast(float x, float eps, float clip) {
    const float kLog2e = 1.4426950216293335f;       // fl(log2 e)
    const float kLog2eLo = 1.9259629911783e-08f;    // log2 e - fl(log2 e)
    const float kLn2 = 0.6931471805599453f;
    x = fminf(fmaxf(x, eps), clip);
    // e^-x = 2^-(hi + lo), hi = fl(x log2e), lo = rounding residue
    float hi = x * kLog2e;
    float lo = fmaf(x, kLog2e, -hi);
    lo = fmaf(x, kLog2eLo, lo);
    float t = ex2_approx(-hi);
    t = fmaf(-t * kLn2, lo, t);  // * (1 - lo ln2)
    // d = 1 - e^-x: Taylor of -expm1(-x) for small x, subtraction otherwise
    float p = fmaf(x, -1.0f / 5040.0f, 1.0f / 720.0f);
    p = fmaf(x, p, -1.0f / 120.0f);
    p = fmaf(x, p, 1.0f / 24.0f);
    p = fmaf(x, p, -1.0f / 6.0f);
    p = fmaf(x, p, 0.5f);
    p = fmaf(x, p, -1.0f);
    float d_small = -x * p;               // x - x^2/2 + x^3/6 - ...
    float d = x < 0.25f ? d_small : 1.0f - t;
    float ratio = (2.0f - d) * rcp_approx(d);
    float phi_log = lg2_approx(ratio) * kLn2;
    // region C: 2 artanh(t)
    float t2 = t * t;
    float s = fmaf(t2, 1.0f / 9.0f, 1.0f / 7.0f);
    s = fmaf(t2, s, 1.0f / 5.0f);
    s = fmaf(t2, s, 1.0f / 3.0f);
    s = fmaf(t2, s, 1.0f);
    float phi_series = 2.0f * t * s;
    return x >= 2.0f ? phi_series : phi_log;
}

}  // namespace qcl
