// kernels.cuh -- device kernels of the layered decoder (sm_100a).
//
// Device layouts.  Codewords are interleaved in groups of W
// lanes (W a power of two <= 32, Bp = G*W >= B, b = g*W + w):
//   llr, posterior L : T[G][n][W]           element (v, b) at (g*n + v)*W + w
//   edge messages R  : T[G][E][z][W]        edge e (slot order), offset k
//   syndrome         : u8[G][S][z][W]       slot order (the reference indexes the
//                                           ORIGINAL row, decoder.py:168-170; the
//                                           upload kernel applies the permutation)
// A thread owns one check (slot s, offset k) for V consecutive lanes w0..w0+V-1.
// Consecutive threads walk (k, w), so for every edge j of the check a warp reads and
// writes one contiguous run of L (variables col*z + (k+shift) mod z are consecutive
// in k) and one contiguous run of R: every access is a coalesced V*sizeof(T)-wide
// vector access and each algorithmic byte crosses the memory system once.
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "phi.cuh"
#include "philox.cuh"

namespace qcl {

// Programmatic dependent launch (sm_90+): no-ops when the grid was launched without the
// programmatic-serialization attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }


constexpr int kBlock = 256;

struct SlotInfo {      // one rearranged row slot of H_compact1
    int32_t edge_off;  // first circulant (slot order)
    int32_t degree;
    int32_t row;       // original base row
    int32_t pad;
};
struct EdgeInfo {      // one circulant of H_compact1
    int32_t var_base;  // base_col * z
    int32_t shift;
    int32_t reused;    // column degree > 1: its posteriors are re-read by later layers
    int32_t pad;
};

// Everything a launch over a contiguous slot range needs.
struct SlotRange {
    const SlotInfo *slots;
    const EdgeInfo *edges;
    int64_t n;        // variables per codeword
    int32_t E;        // circulants
    int32_t S;        // slots (all layers)
    int32_t z;
    const int32_t *slot_list;  // launch unit's slots (nullptr: contiguous from slot0)
    int32_t slot0;    // first slot (or first slot_list entry) of the launch
    int32_t nslots;   // slots in the launch
    int32_t bps;      // blocks per (group, slot)
    int32_t lw;       // log2 W
    int32_t g0;       // first lane group of the launch (groups g0 .. g0 + grid/(nslots*bps) - 1)
};

struct LayerArgs {
    SlotRange r;
    void *L;
    void *R;
    const uint8_t *syn;  // nullptr: all-zero target
    int32_t uniform;     // uniform row degree in the layer (FP64 fold order)
    int32_t clip_r;      // the clip can bind |r| (clip < Phi(eps)); else the r clip is skipped
    const int *n_active; // early termination: skip the launch once every frame converged
    double clip, eps;
    double mag_max;      // FP32 bound on |r|: min(Phi(eps), clip if clip_r)
};

template <typename T, int V> struct Vec;
template <> struct Vec<float, 1> { using type = float; };
template <> struct Vec<float, 2> { using type = float2; };
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<double, 1> { using type = double; };
template <> struct Vec<double, 2> { using type = double2; };

// L2-only (.cg) accesses: state is produced by other CTAs between launches/barriers,
// and nothing is re-read within a layer, so L1 allocation would only risk staleness.
template <typename T, int V>
__device__ __forceinline__ void vload(const T *p, T (&out)[V]) {
    using VT = typename Vec<T, V>::type;
    VT v = __ldcg(reinterpret_cast<const VT *>(p));
    const T *s = reinterpret_cast<const T *>(&v);
#pragma unroll
    for (int i = 0; i < V; i++) out[i] = s[i];
}
template <typename T, int V>
__device__ __forceinline__ void vstore(T *p, const T (&in)[V]) {
    using VT = typename Vec<T, V>::type;
    VT v;
    T *d = reinterpret_cast<T *>(&v);
#pragma unroll
    for (int i = 0; i < V; i++) d[i] = in[i];
    __stcg(reinterpret_cast<VT *>(p), v);
}

__device__ __forceinline__ float clampT(float x, float c) { return fminf(fmaxf(x, -c), c); }
__device__ __forceinline__ double clampT(double x, double c) { return fmin(fmax(x, -c), c); }

template <typename T> __device__ __forceinline__ T phiT(T x, T eps, T clip);
template <> __device__ __forceinline__ float phiT<float>(float x, float eps, float clip) {
    return phi_fast(x, eps, clip);
}
template <> __device__ __forceinline__ double phiT<double>(double x, double eps, double clip) {
    return phi_ref(x, eps, clip);
}

// Phi(|q|) for q already clipped to +-clip: only the eps clamp can bind (the reference
// clamps to [eps, clip] again, decoder.py:104, which is a no-op above eps here).
template <typename T> __device__ __forceinline__ T phi_absq(T q, T eps);
template <> __device__ __forceinline__ float phi_absq<float>(float q, float eps) {
    return phi_fast_ge(fmaxf(fabsf(q), eps));
}
template <> __device__ __forceinline__ double phi_absq<double>(double q, double eps) {
    return log1p(2.0 / expm1(fmax(fabs(q), eps)));
}

// numpy pairwise_sum of a[1..d) (d-1 <= 31 terms), restated for the FP64 parity path:
// fewer than 8 terms is a left fold started from 0.0; otherwise 8 strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail (decoder.py:240,
// np.add.reduceat = a0 + pairwise(rest), measured in SURVEY.md Appendix B P3).
template <int DMAX>
__device__ __forceinline__ double pairwise_rest(const double (&a)[DMAX], int d) {
    const int cnt = d - 1;
    if (cnt < 8) {
        double r = 0.0;
#pragma unroll
        for (int j = 1; j < DMAX; j++)
            if (j < d) r += a[j];
        return r;
    }
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = a[1 + i < DMAX ? 1 + i : 0];
    const int body = cnt - (cnt % 8);
#pragma unroll
    for (int j = 9; j < DMAX; j++)
        if (j - 1 < body) acc[(j - 1) & 7] += a[j];
    double res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
    for (int j = 1; j < DMAX; j++)
        if (j - 1 >= body && j < d) res += a[j];
    return res;
}

// others_j for every edge of a check, in place in ph[j][v].
//   FP32: exclusive prefix + suffix sums (no total - own cancellation);
//   FP64: total - ph_j with the reference's fold order (left fold for a uniform-degree
//         layer, a0 + pairwise(rest) for a ragged one; decoder.py:233, :240).
template <typename T, int V, int D>
__device__ __forceinline__ void others_in_place(T (&ph)[D][V], int d, int uniform) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            T pre = 0, suf = 0, tmp[D];
#pragma unroll
            for (int j = 0; j < D; j++) {
                tmp[j] = pre;
                pre += ph[j][v];
            }
#pragma unroll
            for (int j = D - 1; j >= 0; j--) {
                T p = ph[j][v];
                ph[j][v] = tmp[j] + suf;
                suf += p;
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < V; v++) {
            double col[D];
#pragma unroll
            for (int j = 0; j < D; j++) col[j] = ph[j][v];
            double total;
            if (uniform) {
                total = col[0];
#pragma unroll
                for (int j = 1; j < D; j++)
                    if (j < d) total += col[j];
            } else {
                total = col[0] + pairwise_rest<D>(col, d);
            }
#pragma unroll
            for (int j = 0; j < D; j++) ph[j][v] = total - col[j];
        }
    }
}

// Map blockIdx.x -> (group, slot, k, w0) for a launch over a slot range.
struct Item {
    int g, slot, k, w0;
    bool live;
};
template <int V>
__device__ __forceinline__ Item map_item(const SlotRange &r, int blk = -1) {
    if (blk < 0) blk = blockIdx.x;
    const int chunk = blk % r.bps;
    blk /= r.bps;
    Item it;
    const int si = r.slot0 + blk % r.nslots;
    it.slot = r.slot_list ? r.slot_list[si] : si;
    it.g = r.g0 + blk / r.nslots;
    const int lanes_v = (1 << r.lw) / V;
    const int item = chunk * kBlock + threadIdx.x;
    it.live = item < r.z * lanes_v;
    it.k = item / lanes_v;
    it.w0 = (item - it.k * lanes_v) * V;
    return it;
}

// ---- FP32 check update: tanh rule in sum/difference form -----------------------------
//
// The reference computes r_j = +-Phi(sum_{i != j} Phi(|q_i|)) with Phi(x) = -ln tanh(x/2)
// (decoder.py:225-245).  With u_i = tanh(|q_i|/2) this is the tanh rule (the reference
// test-suite's own check_node_oracle, tests/oracles.py:40-58):
//     |r_j| = 2 artanh(P_j) = ln((1 + P_j) / (1 - P_j)),   P_j = prod_{i != j} u_i.
// Write u_i = (1 - t_i) / (1 + t_i) with t_i = e^{-|q_i|} and, for a set X of edges,
//     A_X = prod (1 + t_i),  B_X = prod (1 - t_i),  S_X = A_X + B_X,  D_X = A_X - B_X,
// so that (1 + P_X) / (1 - P_X) = S_X / D_X.  Up to a common factor 2 (which cancels),
// a single edge is (S, D) = (1, t) and two disjoint sets combine as
//     S = S_X S_Y + D_X D_Y,   D = S_X D_Y + D_X S_Y        (one FMUL + one FFMA each),
// i.e. adding one edge is S' = S + t D, D' = D + t S (two FFMAs).  Every term is
// non-negative: no cancellation anywhere, so D keeps full relative accuracy when every
// other message is strong (D ~ sum t_i, tiny) and S / D -> 1 stays accurate in absolute
// terms when one is weak.  FP32 evaluation per edge: t = 2^(-|q| log2 e) (MUFU.EX2), and
// per output |r_j| = min(lg2(S_j / D_j) ln 2, mag_max) (MUFU.RCP + MUFU.LG2), with
// mag_max = min(Phi(eps), clip if the clip binds r): the reference's clamp of `others` to
// >= eps (decoder.py:104) is exactly |r| <= Phi(eps) (Phi is decreasing and self-
// inverse); its upper clamp at `clip` moves |r| by < Phi(clip) = 1.9e-13.  An input
// |q| < eps gives t = 1, i.e. S = D and r = 0 on the other edges instead of eps = 1e-10.
// 3 MUFU and ~19 instructions per edge (the Phi-domain form needed 6 MUFU and ~37).
// Signs: r_j = |r_j| with sign (q_j < 0) ^ parity(all q < 0) ^ syndrome bit.
//
// QCL_F32_MATH selects how t and |r| are evaluated (the combine is the same):
//   0: MUFU approximations (ex2/rcp/lg2.approx), the fast default;
//   1: libdevice expf / IEEE division / logf (a few ulp end to end), for accuracy A/Bs.
#ifndef QCL_F32_MATH
#define QCL_F32_MATH 0
#endif
#if QCL_F32_MATH == 0
__device__ __forceinline__ float sd_t(float q) { return ex2_approx(fabsf(q) * -1.4426950408889634f); }
__device__ __forceinline__ float sd_mag(float S, float D, float mag_max) {
    // D = 0 only when every other message is infinitely strong: lg2(inf) -> mag_max
    return fminf(lg2_approx(S * rcp_approx(D)) * 0.6931471805599453f, mag_max);
}
#else
__device__ __forceinline__ float sd_t(float q) { return expf(-fabsf(q)); }
__device__ __forceinline__ float sd_mag(float S, float D, float mag_max) {
    return fminf(logf(__fdiv_rn(S, D)), mag_max);
}
#endif

// 16-bit edge messages (QCL_PREC_FP32_MSG16): |r| rounded to FP16 before it is used, so
// the posterior update and the message store see the same value and the next sweep's
// q = L - r_old subtracts exactly what was added
template <bool H>
__device__ __forceinline__ float msg_round(float mag) {
    if constexpr (H) return __half2float(__float2half_rn(mag));
    return mag;
}

// Any degree <= D (edges j >= d are neutral: t = 0, the identity (1, 0) of the combine):
//   in:  q[j][v] = clip(L - r_old), par[v] = syndrome bit
//   out: q[j][v] <- new posterior clip(q + r), ph[j][v] <- new message r
template <int V, int D, bool H = false>
__device__ __forceinline__ void check_update_f32(float (&q)[D][V], float (&ph)[D][V], int (&par)[V], int d,
                                                 float mag_max, float clip) {
#pragma unroll
    for (int v = 0; v < V; v++) {
        float t[D];
#pragma unroll
        for (int j = 0; j < D; j++) {
            if (j < d) {
                t[j] = sd_t(q[j][v]);
                par[v] ^= (q[j][v] < 0.0f);
            } else {
                t[j] = 0.0f;
            }
        }
        float ps = 1.0f, pd = 0.0f, xs[D], xd[D];  // exclusive prefixes
#pragma unroll
        for (int j = 0; j < D; j++) {
            xs[j] = ps;
            xd[j] = pd;
            const float ns = fmaf(t[j], pd, ps);
            pd = fmaf(t[j], ps, pd);
            ps = ns;
        }
        float ss = 1.0f, sd = 0.0f;  // running suffix
#pragma unroll
        for (int j = D - 1; j >= 0; j--) {
            if (j < d) {
                const float S = fmaf(xs[j], ss, xd[j] * sd), Dv = fmaf(xs[j], sd, xd[j] * ss);
                const float mag = msg_round<H>(sd_mag(S, Dv, mag_max));
                const float r = ((q[j][v] < 0.0f) ^ (par[v] != 0)) ? -mag : mag;
                ph[j][v] = r;
                q[j][v] = clampT(q[j][v] + r, clip);
            }
            const float ns = fmaf(t[j], sd, ss);
            sd = fmaf(t[j], ss, sd);
            ss = ns;
        }
    }
}

// Exact degree 4 (the 350 rows of type 3+1 that dominate the MET code): 12 FP32 ops for
// the four exclusive (S, D) pairs, no predication, and signs handled as IEEE sign bits:
// parity = XOR of the q sign bits (^ syndrome), r = |r| | (sign(q) ^ parity).  Exact
// because the FP32 state never holds -0.0 (reset/upload canonicalise it; r != -0.0 and,
// under round-to-nearest, q + r and L - r_old are -0.0 only for -0.0 operands), so the
// sign bit == (q < 0).  Lane pairs use the packed FP32 instructions (FFMA2/FADD2/FMUL2).
template <int V, bool H = false>
__device__ __forceinline__ void check_update_f32_d4(float (&q)[4][V], float (&ph)[4][V], const uint32_t (&synbit)[V],
                                                    float mag_max, float clip) {
#ifndef QCL_PACKED_F32X2
#define QCL_PACKED_F32X2 1
#endif
    if constexpr (QCL_PACKED_F32X2 && QCL_F32_MATH == 0 && V % 2 == 0) {
        // lane pairs on the packed FP32 pipe (FMUL2/FFMA2/FADD2: two IEEE round-to-nearest
        // results per instruction, the same values as the scalar ops below)
#pragma unroll
        for (int v = 0; v < V; v += 2) {
            uint32_t qs[4][2];
            float2 t[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                qs[j][0] = __float_as_uint(q[j][v]) & 0x80000000u;
                qs[j][1] = __float_as_uint(q[j][v + 1]) & 0x80000000u;
                const float2 e = __fmul2_rn(make_float2(fabsf(q[j][v]), fabsf(q[j][v + 1])),
                                            make_float2(-1.4426950408889634f, -1.4426950408889634f));
                t[j] = make_float2(ex2_approx(e.x), ex2_approx(e.y));
            }
            const uint32_t par0 = qs[0][0] ^ qs[1][0] ^ qs[2][0] ^ qs[3][0] ^ synbit[v];
            const uint32_t par1 = qs[0][1] ^ qs[1][1] ^ qs[2][1] ^ qs[3][1] ^ synbit[v + 1];
            const float2 one = make_float2(1.0f, 1.0f);
            const float2 S01 = __ffma2_rn(t[0], t[1], one), D01 = __fadd2_rn(t[0], t[1]);
            const float2 S23 = __ffma2_rn(t[2], t[3], one), D23 = __fadd2_rn(t[2], t[3]);
            float2 S[4], Dv[4];
            S[0] = __ffma2_rn(t[1], D23, S23);
            Dv[0] = __ffma2_rn(t[1], S23, D23);
            S[1] = __ffma2_rn(t[0], D23, S23);
            Dv[1] = __ffma2_rn(t[0], S23, D23);
            S[2] = __ffma2_rn(t[3], D01, S01);
            Dv[2] = __ffma2_rn(t[3], S01, D01);
            S[3] = __ffma2_rn(t[2], D01, S01);
            Dv[3] = __ffma2_rn(t[2], S01, D01);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float2 x = __fmul2_rn(S[j], make_float2(rcp_approx(Dv[j].x), rcp_approx(Dv[j].y)));
                const float2 lg = __fmul2_rn(make_float2(lg2_approx(x.x), lg2_approx(x.y)),
                                             make_float2(0.6931471805599453f, 0.6931471805599453f));
                const float m0 = msg_round<H>(fminf(lg.x, mag_max)), m1 = msg_round<H>(fminf(lg.y, mag_max));
                const float r0 = __uint_as_float(__float_as_uint(m0) | (qs[j][0] ^ par0));
                const float r1 = __uint_as_float(__float_as_uint(m1) | (qs[j][1] ^ par1));
                ph[j][v] = r0;
                ph[j][v + 1] = r1;
                const float2 l = __fadd2_rn(make_float2(q[j][v], q[j][v + 1]), make_float2(r0, r1));
                q[j][v] = clampT(l.x, clip);
                q[j][v + 1] = clampT(l.y, clip);
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < V; v++) {
            uint32_t qs[4];
            float t[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                qs[j] = __float_as_uint(q[j][v]) & 0x80000000u;
                t[j] = sd_t(q[j][v]);
            }
            const uint32_t par = qs[0] ^ qs[1] ^ qs[2] ^ qs[3] ^ synbit[v];
            const float S01 = fmaf(t[0], t[1], 1.0f), D01 = t[0] + t[1];
            const float S23 = fmaf(t[2], t[3], 1.0f), D23 = t[2] + t[3];
            float S[4], Dv[4];
            S[0] = fmaf(t[1], D23, S23);
            Dv[0] = fmaf(t[1], S23, D23);
            S[1] = fmaf(t[0], D23, S23);
            Dv[1] = fmaf(t[0], S23, D23);
            S[2] = fmaf(t[3], D01, S01);
            Dv[2] = fmaf(t[3], S01, D01);
            S[3] = fmaf(t[2], D01, S01);
            Dv[3] = fmaf(t[2], S01, D01);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float mag = msg_round<H>(sd_mag(S[j], Dv[j], mag_max));
                const float r = __uint_as_float(__float_as_uint(mag) | (qs[j] ^ par));
                ph[j][v] = r;
                q[j][v] = clampT(q[j][v] + r, clip);
            }
        }
    }
}

// FP64 parity update (reference formula and fold order), same in/out convention.
template <int V, int D>
__device__ __forceinline__ void check_update_f64(double (&q)[D][V], double (&ph)[D][V], int (&par)[V], int d,
                                                 double eps, double clip, int uniform) {
#pragma unroll
    for (int j = 0; j < D; j++) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            if (j < d) {
                ph[j][v] = phi_absq<double>(q[j][v], eps);
                par[v] ^= (q[j][v] < 0.0);
            } else {
                ph[j][v] = 0.0;
            }
        }
    }
    others_in_place<double, V, D>(ph, d, uniform);
#pragma unroll
    for (int j = 0; j < D; j++) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            if (j < d) {
                const double mag = phi_ref(ph[j][v], eps, clip);
                const double r = clampT(((q[j][v] < 0.0) ^ (par[v] != 0)) ? -mag : mag, clip);
                ph[j][v] = r;
                q[j][v] = clampT(q[j][v] + r, clip);
            }
        }
    }
}

template <int V, int D>
__device__ __forceinline__ void check_update(float (&q)[D][V], float (&ph)[D][V], int (&par)[V], int d,
                                             const LayerArgs &a) {
    if constexpr (D == 4) {
        if (d == 4) {  // warp-uniform: a unit's slots share the degree class
            uint32_t sb[V];
#pragma unroll
            for (int v = 0; v < V; v++) sb[v] = (uint32_t)par[v] << 31;
            check_update_f32_d4<V>(q, ph, sb, (float)a.mag_max, (float)a.clip);
            return;
        }
    }
    check_update_f32<V, D>(q, ph, par, d, (float)a.mag_max, (float)a.clip);
}
template <int V, int D>
__device__ __forceinline__ void check_update(double (&q)[D][V], double (&ph)[D][V], int (&par)[V], int d,
                                             const LayerArgs &a) {
    check_update_f64<V, D>(q, ph, par, d, a.eps, a.clip, a.uniform);
}

// One layered update of every check in the launch's slot range, for every group
// (decoder.py:212-250, _layer_update_core).  Rows of one merged layer touch disjoint
// columns (checked at plan creation, decoder.py:144-154), so the read-modify-write of
// L is race free.  Offsets inside a lane group are 32-bit (n*W and E*z*W < 2^31).
template <typename T, int V, int DMAX, bool HAS_SYN>
__device__ __forceinline__ void layer_tile(const LayerArgs &a, const Item &it, const SlotInfo &si,
                                           const EdgeInfo *s_edge);

template <typename T, int V, int DMAX, bool HAS_SYN>
__global__ void __launch_bounds__(kBlock) layer_kernel(LayerArgs a) {
    // programmatic dependent launch (qcldpc.cu launch_pdl): the next layer's grid may start
    // now; this one's prologue (immutable plan tables) overlaps the previous layer's tail,
    // and every read of state the previous kernels wrote follows griddepcontrol.wait
    pdl_launch_dependents();
    __shared__ EdgeInfo s_edge[DMAX];
    const Item it = map_item<V>(a.r);
    const SlotInfo si = a.r.slots[it.slot];
    const int d = si.degree;
    if (threadIdx.x < d) s_edge[threadIdx.x] = a.r.edges[si.edge_off + threadIdx.x];
    pdl_wait();
    if (a.n_active && *(volatile const int *)a.n_active == 0) return;
    __syncthreads();
    if (!it.live) return;
    layer_tile<T, V, DMAX, HAS_SYN>(a, it, si, s_edge);
}

// The update of one thread's check(s) (decoder.py:212-250): shared by the per-layer
// kernel above and the persistent single-launch kernel below.
template <typename T, int V, int DMAX, bool HAS_SYN>
__device__ __forceinline__ void layer_tile(const LayerArgs &a, const Item &it, const SlotInfo &si,
                                           const EdgeInfo *s_edge) {
    const int d = si.degree;
    const int z = a.r.z, lw = a.r.lw, k = it.k;
    T *Lg = reinterpret_cast<T *>(a.L) + (((size_t)it.g * a.r.n) << lw) + it.w0;
    T *Rg = reinterpret_cast<T *>(a.R) + (((((size_t)it.g * a.r.E + si.edge_off) * z) + k) << lw) + it.w0;
    const T clip = (T)a.clip;

    T q[DMAX][V], ph[DMAX][V];
    uint32_t loff[DMAX];
    int par[V];
    if (HAS_SYN) {
        const uint8_t *sp = a.syn + ((((int64_t)it.g * a.r.S + it.slot) * z + k) << lw) + it.w0;
#pragma unroll
        for (int i = 0; i < V; i++) par[i] = sp[i] & 1;
    } else {
#pragma unroll
        for (int i = 0; i < V; i++) par[i] = 0;
    }
    // gather: all 2d loads issued before any use (memory-level parallelism)
#pragma unroll
    for (int j = 0; j < DMAX; j++) {
        if (j < d) {
            int pos = k + s_edge[j].shift;
            pos -= (pos >= z) ? z : 0;
            loff[j] = (uint32_t)(s_edge[j].var_base + pos) << lw;
            T lv[V], rv[V];
            vload<T, V>(Lg + loff[j], lv);
            vload<T, V>(Rg + ((uint32_t)(j * z) << lw), rv);
#pragma unroll
            for (int i = 0; i < V; i++) q[j][i] = clampT(lv[i] - rv[i], clip);
        } else {
#pragma unroll
            for (int i = 0; i < V; i++) q[j][i] = (T)0;
        }
    }
    check_update<V, DMAX>(q, ph, par, d, a);
    // scatter
#pragma unroll
    for (int j = 0; j < DMAX; j++) {
        if (j < d) {
            vstore<T, V>(Rg + ((uint32_t)(j * z) << lw), ph[j]);
            vstore<T, V>(Lg + loff[j], q[j]);
        }
    }
}

// ---- persistent per-layer engine for one or two codewords (BASELINE configs[1]) -------
// With W <= 2 lanes every layer is a few hundred CTAs of dependent work, and a decode is
// ~1650 dependent layer launches whose launch gaps set the latency (PDL hides part of
// it).  Here the whole decode is ONE cooperative launch: every CTA walks the launch units
// of a sweep in schedule order (decoder.py:259-262), takes the blocks b = blockIdx.x,
// blockIdx.x + gridDim.x, ... of each unit (the same check-to-thread map and the same
// layer_tile arithmetic as layer_kernel, so results are bit-identical to it), and a
// grid barrier separates consecutive units (layer l + 1 reads what layer l wrote).
struct alignas(16) PersistUnit {
    LayerArgs a;
    int32_t blocks;  // G * nslots * bps
    int32_t dcls;    // DMAX bucket of the unit: 4, 8, 12, 16 or 32
    int32_t layer;   // merged layer (units of one layer touch disjoint columns: no barrier)
};
struct PersistArgs {
    const PersistUnit *units;  // [nu] one sweep, schedule order
    int32_t nu, sweeps;
    int32_t S, E, nlist;       // plan tables copied to shared memory at kernel start
    const SlotInfo *slots;
    const EdgeInfo *edges;
    const int32_t *slot_list;
    unsigned *bar;             // [0] completed barriers, [32] arrivals, [32 (5 + cta)] per-CTA arrivals
                               // (zeroed before the launch)
    const int *n_active;       // early termination: skip the launch once every frame converged
    int32_t bar_mode;          // persist_grid_barrier
};
static_assert(sizeof(PersistUnit) % 16 == 0, "PersistUnit is copied in 16-byte words");
__host__ __device__ constexpr size_t persist_smem_bytes(int nu, int S, int E, int nlist) {
    return sizeof(PersistUnit) * nu + sizeof(SlotInfo) * S + sizeof(EdgeInfo) * E + sizeof(int32_t) * nlist;
}

// Barrier k of the launch (bar.sync orders each CTA's global stores before its thread-0
// release -- cumulativity -- and the acquire polls order the next unit's loads after every
// CTA's stores).  Modes (PersistArgs::bar_mode, QCL_PERSIST_BAR):
//   0: one acq_rel atomic arrival per CTA; the CTA whose arrival completes the count
//      releases the barrier word (a separate line) that the others poll;
//   1: fire-and-forget release reductions, every CTA polls the arrival counter;
//   2: per-CTA arrival flags (one line each) gathered by CTA 0, which releases the word.
// Single codeword, 50 iterations (tools/persist_sweep.sh): 1 = 4.44 ms, 0 = 5.31, 2 = 6.10;
// a 32 ns poll back-off (4.53) and arrivals spread over four lines (5.82) were slower.
constexpr int kPersistThreads = 512;  // at most two 256-check blocks per CTA
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void persist_grid_barrier(unsigned *bar, unsigned k, int mode) {
    __syncthreads();
    if (mode == 2) {
        if (threadIdx.x == 0) st_release_u32(bar + 32 * (5 + blockIdx.x), k);
        if (blockIdx.x == 0) {
            for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x)
                while (ld_acquire_u32(bar + 32 * (5 + c)) < k) {
                }
            __syncthreads();
            if (threadIdx.x == 0) st_release_u32(bar, k);
        } else if (threadIdx.x == 0) {
            while (ld_acquire_u32(bar) < k) {
            }
        }
    } else if (threadIdx.x == 0) {
        if (mode == 1) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 32) : "memory");
            while (ld_acquire_u32(bar + 32) < k * gridDim.x) {
            }
        } else {
            unsigned old;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 32) : "memory");
            if (old == k * gridDim.x - 1)
                st_release_u32(bar, k);
            else
                while (ld_acquire_u32(bar) < k) {
                }
        }
    }
    __syncthreads();
}

template <typename T, bool HAS_SYN, int MAXD>  // MAXD: the largest unit bucket of the plan
__global__ void __launch_bounds__(kPersistThreads, 1) layer_persist_kernel(PersistArgs pa) {
    extern __shared__ __align__(16) unsigned char psm[];
    PersistUnit *units = reinterpret_cast<PersistUnit *>(psm);
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(units + pa.nu);
    EdgeInfo *edges = reinterpret_cast<EdgeInfo *>(slots + pa.S);
    int32_t *slist = reinterpret_cast<int32_t *>(edges + pa.E);
    if (pa.n_active && *(volatile const int *)pa.n_active == 0) return;  // uniform: set between launches
    {
        const int4 *src = reinterpret_cast<const int4 *>(pa.units);
        int4 *dst = reinterpret_cast<int4 *>(units);
        for (int i = threadIdx.x; i < (int)(sizeof(PersistUnit) / 16) * pa.nu; i += blockDim.x) dst[i] = src[i];
        for (int i = threadIdx.x; i < pa.S; i += blockDim.x) slots[i] = pa.slots[i];
        for (int i = threadIdx.x; i < pa.E; i += blockDim.x) edges[i] = pa.edges[i];
        for (int i = threadIdx.x; i < pa.nlist; i += blockDim.x) slist[i] = pa.slot_list[i];
    }
    __syncthreads();
    unsigned k = 0;
    for (int t = 0; t < pa.sweeps; t++) {
        for (int u = 0; u < pa.nu; u++) {
            const PersistUnit &pu = units[u];
            const SlotRange &r = pu.a.r;
            const int nb = pu.blocks, dc = pu.dcls;
            const int halves = blockDim.x / kBlock;
            const int tid = threadIdx.x % kBlock;
            for (int b = blockIdx.x * halves + threadIdx.x / kBlock; b < nb; b += gridDim.x * halves) {
                // map_item<1> with the slot list in shared memory
                const int chunk = b % r.bps, blk = b / r.bps;
                Item it;
                it.slot = slist[r.slot0 + blk % r.nslots];
                it.g = r.g0 + blk / r.nslots;
                const int item = chunk * kBlock + tid;
                it.live = item < (r.z << r.lw);
                it.k = item >> r.lw;
                it.w0 = item - (it.k << r.lw);
                if (!it.live) continue;
                const SlotInfo si = slots[it.slot];
                const EdgeInfo *se = edges + si.edge_off;
                if (dc == 4)
                    layer_tile<T, 1, 4, HAS_SYN>(pu.a, it, si, se);
                else if (MAXD >= 8 && dc == 8)
                    layer_tile<T, 1, (MAXD >= 8 ? 8 : 4), HAS_SYN>(pu.a, it, si, se);
                else if (MAXD >= 12 && dc == 12)
                    layer_tile<T, 1, (MAXD >= 12 ? 12 : 4), HAS_SYN>(pu.a, it, si, se);
                else if (MAXD >= 16 && dc == 16)
                    layer_tile<T, 1, (MAXD >= 16 ? 16 : 4), HAS_SYN>(pu.a, it, si, se);
                else if (MAXD >= 32)
                    layer_tile<T, 1, (MAXD >= 32 ? 32 : 4), HAS_SYN>(pu.a, it, si, se);
            }
            if (u + 1 < pa.nu && units[u + 1].layer == pu.layer) continue;  // same layer: disjoint columns
            persist_grid_barrier(pa.bar, ++k, pa.bar_mode);
        }
    }
}

// ---- hard decisions and syndrome check on packed sign words ------------------------
// signs[g][v]: bit w = (L[g][v][w] < 0) -- one uint32 per variable carries the hard
// decisions of all W lanes (decoder.py:264-266; -0.0 decides to 0 like `< 0`).
// Lane groups whose frames have all converged (early termination) are skipped when
// gact != nullptr: their outputs were frozen at convergence, so nothing observable
// depends on their later state.
// Sign word of variable v of group g (element i = g*n + v): bit w = (L[g][v][w] < 0).
template <typename T>
__device__ __forceinline__ uint32_t sign_word(const T *L, int64_t i, int lw) {
    const int W = 1 << lw;
    const T *p = L + (i << lw);
    uint32_t m = 0;
    if (sizeof(T) == 4 && (W & 3) == 0) {
        for (int w = 0; w < W; w += 4) {
            const float4 x = __ldcg(reinterpret_cast<const float4 *>(p + w));
            m |= ((uint32_t)(x.x < 0.0f) | ((uint32_t)(x.y < 0.0f) << 1) | ((uint32_t)(x.z < 0.0f) << 2) |
                  ((uint32_t)(x.w < 0.0f) << 3)) << w;
        }
    } else {
        for (int w = 0; w < W; w++) m |= (uint32_t)(__ldcg(p + w) < (T)0) << w;
    }
    return m;
}

// signs[v][g]: bit w = (L[g][v][w] < 0), i.e. all lane groups of a variable side by side,
// so one syndrome-check thread reads every group's sign word of a variable in one go.
template <typename T>
__global__ void __launch_bounds__(kBlock) sign_pack_kernel(const T *L, int64_t Gn, int lw, uint32_t *signs, int64_t n,
                                                           const uint8_t *gact) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over G * n: one variable of one group
    const int64_t g = i < Gn ? i / n : -1, v = i - g * n;
    const bool live = i < Gn && (!gact || gact[g]);
    if (!live) return;
    const uint32_t m = sign_word(L, i, lw);
    signs[v * (Gn / n) + g] = m;
}

// The same, one thread per variable over all lane groups: no 64-bit division per thread,
// and each thread writes its variable's G sign words contiguously (chunks of 4 groups as
// one 16-byte store when G % 4 == 0).
template <typename T>
__global__ void __launch_bounds__(kBlock) sign_pack_var_kernel(const T *L, int G, int lw, uint32_t *signs, int64_t n,
                                                               const uint8_t *gact) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint32_t *out = signs + v * G;
    if ((G & 3) == 0) {
        for (int g = 0; g < G; g += 4) {
            const bool a0 = !gact || gact[g], a1 = !gact || gact[g + 1], a2 = !gact || gact[g + 2],
                       a3 = !gact || gact[g + 3];
            if (!(a0 | a1 | a2 | a3)) continue;
            uint4 m;
            m.x = a0 ? sign_word(L, (int64_t)g * n + v, lw) : out[g];
            m.y = a1 ? sign_word(L, (int64_t)(g + 1) * n + v, lw) : out[g + 1];
            m.z = a2 ? sign_word(L, (int64_t)(g + 2) * n + v, lw) : out[g + 2];
            m.w = a3 ? sign_word(L, (int64_t)(g + 3) * n + v, lw) : out[g + 3];
            *reinterpret_cast<uint4 *>(out + g) = m;
        }
    } else {
        for (int g = 0; g < G; g++)
            if (!gact || gact[g]) out[g] = sign_word(L, (int64_t)g * n + v, lw);
    }
}

// gact[g] = some frame of lane group g is still active (early termination).
__global__ void group_active_kernel(int64_t Bp, int lw, const uint8_t *active, uint8_t *gact) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if ((g << lw) >= Bp) return;
    uint8_t any = 0;
    for (int w = 0; w < (1 << lw); w++) any |= active[(g << lw) + w];
    gact[g] = any;
}

// Syndrome bytes (lanes layout) -> one uint32 of W lane bits per check.
// Syndrome bytes (lanes layout u8[G][S][z][W]) -> packed[(s*z + k)*G + g], W lane bits.
__global__ void syn_pack_kernel(const uint8_t *syn, int64_t words, int lw, int64_t Sz, uint32_t *packed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over G * S * z, (g, check)
    if (i >= words) return;
    const int W = 1 << lw;
    const int64_t G = words / Sz, g = i / Sz, c = i - g * Sz;
    uint32_t v = 0;
    for (int w = 0; w < W; w++) v |= (uint32_t)(syn[(i << lw) + w] & 1) << w;
    packed[c * G + g] = v;
}

// syndrome_satisfied (decoder.py:268-273) for all lanes at once: one thread per check
// (s, k) covers every lane group: XOR of the d variables' sign words (^ packed target
// syndrome); a set bit marks that lane's codeword unsatisfied.  Lanes OR-reduce per
// group before one atomic.  Groups in chunks of 8 (two 16-byte loads per variable).
__global__ void __launch_bounds__(kBlock) check_packed_kernel(const SlotInfo *slots, const EdgeInfo *edges,
                                                              int64_t n, int S, int z, int G,
                                                              const uint32_t *signs, const uint32_t *synpack,
                                                              uint32_t *unsat_mask, const uint8_t *gact) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // over S * z checks (< 2^31)
    const uint32_t total = (uint32_t)S * (uint32_t)z;
    const bool live = i < total;
    const uint32_t s = live ? i / (uint32_t)z : 0, k = live ? i - s * (uint32_t)z : 0;
    const SlotInfo si = live ? slots[s] : SlotInfo{0, 0, 0, 0};
    const bool vec = (G & 3) == 0;
    for (int g0 = 0; g0 < G; g0 += 8) {
        bool any_active = true;
        if (gact) {
            any_active = false;
            for (int c = 0; c < 8 && g0 + c < G; c++) any_active |= gact[g0 + c] != 0;
        }
        if (!any_active) continue;  // warp-uniform: every frame of these groups converged
        uint32_t p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int cnt = min(8, G - g0);
        if (live) {
            if (synpack)
                for (int c = 0; c < cnt; c++) p[c] = synpack[(int64_t)i * G + g0 + c];
            for (int j = 0; j < si.degree; j++) {
                const EdgeInfo e = edges[si.edge_off + j];
                int pos = (int)k + e.shift;
                pos -= (pos >= z) ? z : 0;
                const uint32_t *row = signs + (int64_t)(e.var_base + pos) * G + g0;
                if (vec && cnt == 8) {
                    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(row));
                    const uint4 b = __ldg(reinterpret_cast<const uint4 *>(row) + 1);
                    p[0] ^= a.x; p[1] ^= a.y; p[2] ^= a.z; p[3] ^= a.w;
                    p[4] ^= b.x; p[5] ^= b.y; p[6] ^= b.z; p[7] ^= b.w;
                } else {
                    for (int c = 0; c < cnt; c++) p[c] ^= __ldg(row + c);
                }
            }
        }
        // warp OR-reduce, then block OR in shared memory: one global atomic per group and
        // block (same-address global atomics from every warp serialise in L2)
        __shared__ uint32_t s_acc[8];
        if (threadIdx.x < 8) s_acc[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const uint32_t any = __reduce_or_sync(0xffffffffu, p[c]);
            if (any && (threadIdx.x & 31) == 0) atomicOr(&s_acc[c], any);
        }
        __syncthreads();
        if (threadIdx.x < 8 && g0 + (int)threadIdx.x < G && s_acc[threadIdx.x])
            atomicOr(unsat_mask + g0 + threadIdx.x, s_acc[threadIdx.x]);
        __syncthreads();
    }
}

// Words (B, n) from packed signs for the codewords with take[b] (all if take == nullptr).
// One thread per variable loops over the codewords: a pass that takes nothing (the
// common early-termination iteration) costs n/256 blocks reading B flags.
__global__ void __launch_bounds__(kBlock) words_from_signs_kernel(const uint32_t *signs, int64_t n, int lw,
                                                                  int64_t B, const uint8_t *take, uint8_t *words) {
    const int64_t G = (B + (1 << lw) - 1) >> lw;
    if (take) {  // most early-termination sweeps take no frame: the whole block exits
        __shared__ int s_any;
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        for (int64_t b = threadIdx.x; b < B; b += blockDim.x)
            if (take[b]) s_any = 1;
        __syncthreads();
        if (!s_any) return;
    }
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int Wm = (1 << lw) - 1;
    for (int64_t b = 0; b < B; b++) {
        if (take && !take[b]) continue;
        words[b * n + v] = (uint8_t)((__ldg(signs + v * G + (b >> lw)) >> (b & Wm)) & 1u);
    }
}

// Fused early termination (flow.cuh): active-lane masks at the start of a decode, and the
// words afterwards -- a converged codeword's lane bits frozen at its convergence (fsign),
// any other's from the hard-decision snapshot of the last sweep (decoder.py:307-311).
__global__ void amask_init_kernel(int G, int lw, int64_t B, uint32_t *amask) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const int64_t live = B - ((int64_t)g << lw);
    const int W = 1 << lw;
    amask[g] = live >= W ? (W == 32 ? 0xffffffffu : (1u << W) - 1u) : live <= 0 ? 0u : (1u << live) - 1u;
}

// Snapshot lane bits (both sweep parities) of the variables of columns no row touches.
__global__ void snap_untouched_kernel(const float *L, const int32_t *cols, int ncols, int z, int64_t n, int G,
                                      int lw, uint8_t *snap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_g = (int64_t)ncols * z;
    if (i >= per_g * G) return;
    const int64_t g = i / per_g, r = i - g * per_g;
    const int64_t v = (int64_t)cols[r / z] * z + r % z;
    const int W = 1 << lw;
    uint32_t bits = 0;
    for (int w = 0; w < W; w++) bits |= (uint32_t)(L[((g * n + v) << lw) + w] < 0.0f) << w;
    snap[g * n + v] = (uint8_t)bits;
    snap[((int64_t)G + g) * n + v] = (uint8_t)bits;
}

__global__ void __launch_bounds__(kBlock) et_words_kernel(const uint8_t *snap_last, const uint8_t *fsign,
                                                          const uint8_t *conv, int64_t n, int lw, int64_t B,
                                                          uint8_t *words) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int Wm = (1 << lw) - 1;
    for (int64_t b = 0; b < B; b++) {
        const uint8_t *src = conv[b] ? fsign : snap_last;
        words[b * n + v] = (uint8_t)((src[(b >> lw) * n + v] >> (b & Wm)) & 1u);
    }
}

__device__ __forceinline__ uint8_t lane_unsat(const uint32_t *mask, int64_t b, int lw) {
    return (uint8_t)((mask[b >> lw] >> (b & ((1 << lw) - 1))) & 1u);
}

// Early-termination bookkeeping after sweep t (decoder.py:295-305): codewords whose
// hard decision satisfies the syndrome for the first time freeze words/iterations.
__global__ void et_update_kernel(int64_t B, int t, const uint32_t *unsat_mask, int lw, uint8_t *active,
                                 uint8_t *take, uint8_t *converged, int64_t *iterations, int *n_active) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    uint8_t newly = active[b] && !lane_unsat(unsat_mask, b, lw);
    take[b] = newly;
    if (newly) {
        active[b] = 0;
        converged[b] = 1;
        iterations[b] = t;
        atomicSub(n_active, 1);
    }
}

// End of decode for codewords still active (decoder.py:307-311).
__global__ void finalize_kernel(int64_t B, const uint32_t *unsat_mask, int lw, const uint8_t *active, uint8_t *take,
                                uint8_t *converged) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    take[b] = active[b];
    if (active[b]) converged[b] = !lane_unsat(unsat_mask, b, lw);
}

__global__ void decode_init_kernel(int64_t B, int64_t Bp, int max_iter, uint8_t *active, uint8_t *converged,
                                   int64_t *iterations, int *n_active) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0) *n_active = (int)B;
    if (b >= Bp) return;
    active[b] = b < B;
    if (b < B) {
        converged[b] = 0;
        iterations[b] = max_iter;
    }
}

// Host (B, n) LLRs (f64 or f32) -> T[G][n][W], rows b >= B zero-filled.
template <typename T, typename S>
__global__ void llr_to_lanes_kernel(const S *src, int64_t B, int64_t Bp, int64_t n, int lw, T *dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over Bp * n, lane fastest
    if (i >= Bp * n) return;
    const int W = 1 << lw;
    int64_t w = i & (W - 1);
    int64_t rest = i >> lw;
    int64_t v = rest % n, g = rest / n;
    int64_t b = (g << lw) + w;
    dst[i] = b < B ? (T)src[b * n + v] : (T)0;
}

// posterior = clip(llr), messages = 0 (new_state, decoder.py:191-202).  For the FP32
// path the clip is applied in FP64 before the cast (inputs may be +-inf).
// The "+ 0" maps -0.0 to +0.0 (same decision: -0.0 < 0 is false, decoder.py:266); the
// FP32 kernels rely on the state never holding -0.0 (check_update_f32_d4).
template <typename T>
__global__ void reset_kernel(const T *llr, T *L, int64_t count, double clip) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (sizeof(T) == 4) {  // four values per thread (16-byte accesses); count % 4 == 0 (W >= 4)
        if ((count & 3) == 0) {
            if (4 * i >= count) return;
            float4 x = reinterpret_cast<const float4 *>(llr)[i];
            x.x = (float)clampT((double)x.x, clip) + 0.0f;
            x.y = (float)clampT((double)x.y, clip) + 0.0f;
            x.z = (float)clampT((double)x.z, clip) + 0.0f;
            x.w = (float)clampT((double)x.w, clip) + 0.0f;
            reinterpret_cast<float4 *>(L)[i] = x;
            return;
        }
    }
    if (i < count) L[i] = (T)clampT((double)llr[i], clip) + (T)0;
}

// Reference-layout FP64 state <-> lanes.  post (B, n); msg (B, E*z) [e][k].
template <typename T, typename RT = T>
__global__ void state_in_kernel(const double *post, const double *msg, int64_t B, int64_t n, int64_t Ez,
                                int lw, T *L, RT *R, int64_t Bp) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int W = 1 << lw;
    int64_t w = i & (W - 1), rest = i >> lw;
    if (i < Bp * n) {
        int64_t v = rest % n, g = rest / n, b = (g << lw) + w;
        L[i] = b < B ? (T)post[b * n + v] + (T)0 : (T)0;  // + 0: no -0.0 in the state
    }
    if (i < Bp * Ez) {
        int64_t x = rest % Ez, g = rest / Ez, b = (g << lw) + w;
        if constexpr (sizeof(RT) == 2)  // one rounding, double -> FP16
            R[i] = __double2half((b < B && msg) ? msg[b * Ez + x] + 0.0 : 0.0);
        else
            R[i] = (b < B && msg) ? (T)msg[b * Ez + x] + (T)0 : (T)0;
    }
}
__device__ __forceinline__ double msg_f64(double x) { return x; }
__device__ __forceinline__ double msg_f64(float x) { return (double)x; }
__device__ __forceinline__ double msg_f64(__half x) { return (double)__half2float(x); }
template <typename T, typename RT = T>
__global__ void state_out_kernel(const T *L, const RT *R, int64_t B, int64_t n, int64_t Ez, int lw,
                                 double *post, double *msg) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over B * max(n, Ez), row-major
    int64_t b = i / (n > Ez ? n : Ez), x = i % (n > Ez ? n : Ez);
    if (b >= B) return;
    const int W = 1 << lw;
    int64_t g = b >> lw, w = b & (W - 1);
    if (post && x < n) post[b * n + x] = (double)L[((g * n + x) << lw) + w];
    if (msg && x < Ez) msg[b * Ez + x] = msg_f64(R[((g * Ez + x) << lw) + w]);
}

// Target syndrome (B, m) in original row order -> u8[G][S][z][W] in slot order.
__global__ void syndrome_to_lanes_kernel(const uint8_t *src, const SlotInfo *slots, int64_t B, int64_t Bp,
                                         int S, int z, int lw, uint8_t *dst, int *any_set) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over Bp * S * z
    if (i >= Bp * (int64_t)S * z) return;
    const int W = 1 << lw;
    int64_t w = i & (W - 1), rest = i >> lw;
    int64_t k = rest % z;
    rest /= z;
    int64_t s = rest % S, g = rest / S, b = (g << lw) + w;
    const int64_t m = (int64_t)S * z;
    const uint8_t bit = b < B ? (src[b * m + (int64_t)slots[s].row * z + k] != 0) : 0;
    dst[i] = bit;
    if (bit) *any_set = 1;  // benign race: every writer stores 1
}

// Syndrome (lanes layout) of words (B, n) -- encode mode target H*c (bench.py:225-226).
__global__ void __launch_bounds__(kBlock) syndrome_of_words_kernel(SlotRange r, const uint8_t *words,
                                                                   int64_t B, uint8_t *syn) {
    const Item it = map_item<1>(r);
    if (!it.live) return;
    const SlotInfo si = r.slots[it.slot];
    const int64_t b = ((int64_t)it.g << r.lw) + it.w0;
    int p = 0;
    if (b < B) {
        for (int j = 0; j < si.degree; j++) {
            EdgeInfo e = r.edges[si.edge_off + j];
            int pos = it.k + e.shift;
            pos -= (pos >= r.z) ? r.z : 0;
            p ^= words[b * r.n + e.var_base + pos] & 1;
        }
    }
    syn[((((int64_t)it.g * r.S + it.slot) * r.z + it.k) << r.lw) + it.w0] = (uint8_t)p;
}

// Device BIAWGN channel (channel.py:41-56 semantics): frame b of the state is frame
// first_frame + b; LLR = 2 (1 - 2c + sigma n) / sigma^2 written straight into the lanes
// layout.  One thread = 4 consecutive variables of one frame (one Philox block).
template <typename T>
__global__ void synth_llr_kernel(int64_t B, int64_t Bp, int64_t n, int lw, uint64_t seed, uint32_t snr_idx,
                                 int64_t first_frame, double sigma, double sigma2, int encode,
                                 T *llr, uint8_t *truths) {
    const int64_t quads = (n + 3) / 4;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // lane fastest
    if (i >= Bp * quads) return;
    const int W = 1 << lw;
    int64_t w = i & (W - 1), rest = i >> lw;
    int64_t qv = rest % quads, g = rest / quads, b = (g << lw) + w;
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const uint64_t frame = (uint64_t)(first_frame + b);
    u32x4 ctr{(uint32_t)qv, (uint32_t)frame, (uint32_t)(frame >> 32), snr_idx & 0x7fffffffu};
    double nz[4];
    normals4(philox4x32_10(ctr, k0, k1), nz);
    uint32_t cbits = 0;
    if (encode) {
        u32x4 c2 = ctr;
        c2.w |= 0x80000000u;
        u32x4 rb = philox4x32_10(c2, k0, k1);
        cbits = (rb.x & 1) | ((rb.y & 1) << 1) | ((rb.z & 1) << 2) | ((rb.w & 1) << 3);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
        int64_t v = qv * 4 + j;
        if (v >= n) break;
        int c = (cbits >> j) & 1;
        double r = (1.0 - 2.0 * c) + sigma * nz[j];
        double val = b < B ? 2.0 * r / sigma2 : 0.0;
        llr[((g * n + v) << lw) + w] = (T)val;
        if (truths && b < B) truths[b * n + v] = (uint8_t)c;
    }
}

// Campaign frame errors (bench.py:236-237): mismatch[b] = 1 when the decoded word of
// frame b differs anywhere from its transmitted word (all-zero when truths == nullptr).
// blockIdx.y = frame; 16-byte vector compares when n is a multiple of 16.
__global__ void __launch_bounds__(kBlock) frame_mismatch_kernel(const uint8_t *words, const uint8_t *truths,
                                                                int64_t n, int64_t B, uint8_t *mismatch) {
    // frames grid-stride along y (gridDim.y is capped at 65535)
    for (int64_t b = blockIdx.y; b < B; b += gridDim.y) {
        const uint8_t *w = words + b * n;
        const uint8_t *t = truths ? truths + b * n : nullptr;
        bool bad = false;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        if ((n & 15) == 0) {
            const uint4 *w4 = reinterpret_cast<const uint4 *>(w);
            const uint4 *t4 = reinterpret_cast<const uint4 *>(t);
            for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 16; i += stride) {
                const uint4 x = __ldg(w4 + i);
                const uint4 y = t ? __ldg(t4 + i) : make_uint4(0, 0, 0, 0);
                bad |= ((x.x ^ y.x) | (x.y ^ y.y) | (x.z ^ y.z) | (x.w ^ y.w)) != 0;
            }
        } else {
            for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
                bad |= w[i] != (t ? t[i] : 0);
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0) mismatch[b] = 1;
    }
}

// ---- frame pool (qcl_state_decode_pool): lanes refilled as their frames finish --------
//
// Campaign decodes with early termination run a stream of frames through the lanes of one
// state: a lane whose frame converged (or hit the iteration cap) records the frame's
// outcome and takes the next frame, so a batch no longer runs to the cap for one slow
// frame.  Per-frame outcomes are unchanged: frames are independent, every frame runs the
// same layered sweeps from its own new_state (a refilled lane starts from L = clip(llr),
// and the flow kernel treats its old messages as zero in its first sweep).

// lane_any[g] |= bit w when the hard decision of lane w of group g has any bit set (the
// all-zero word is the transmitted one: a converged frame is in error iff a bit is set).
// Grid-stride over variables (variable-major sign words, G per variable), per-thread OR
// accumulators, then warp and block reductions: one atomic per group and block.
__global__ void __launch_bounds__(kBlock) lane_any_kernel(const uint32_t *signs, int64_t n, int G,
                                                          const uint8_t *gact, uint32_t *lane_any) {
    __shared__ uint32_t s_acc[32];
    for (int g0 = 0; g0 < G; g0 += 32) {
        const int cnt = min(32, G - g0);
        if (threadIdx.x < 32) s_acc[threadIdx.x] = 0;
        __syncthreads();
        uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c0 = 0; c0 < cnt; c0 += 8) {
            for (int c = 0; c < 8; c++) acc[c] = 0;
            for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
                const uint32_t *row = signs + v * G + g0 + c0;
#pragma unroll
                for (int c = 0; c < 8; c++)
                    if (c0 + c < cnt) acc[c] |= __ldg(row + c);
            }
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const uint32_t m = __reduce_or_sync(0xffffffffu, acc[c]);
                if (m && (threadIdx.x & 31) == 0) atomicOr(&s_acc[c0 + c], m);
            }
        }
        __syncthreads();
        if ((int)threadIdx.x < cnt && s_acc[threadIdx.x] && (!gact || gact[g0 + threadIdx.x]))
            atomicOr(lane_any + g0 + threadIdx.x, s_acc[threadIdx.x]);
        __syncthreads();
    }
}

// After sweep t: per lane, count the sweep, and finish the frame when its syndrome is met or
// the cap is reached (outcome recorded at its frame index); hand the lane the next frame
// (fresh for the next sweep, queued for the refill kernel) or retire it.
__global__ void pool_update_kernel(int64_t Bp, int lw, int max_iter, const uint32_t *unsat_mask,
                                   const uint32_t *lane_any, int64_t first_frame, int64_t n_frames,
                                   int64_t *lane_frame, int32_t *lane_iter, uint8_t *active, int *n_active,
                                   uint8_t *out_conv, int64_t *out_iters, uint8_t *out_err, int32_t *counts,
                                   int32_t *refill, uint32_t *fresh, int *claim) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0) {  // the next sweep: its index (counts[2], read by the flow kernel) and claim counter
        counts[2]++;
        *claim = 0;
    }
    if (b >= Bp) return;
    const int64_t f = lane_frame[b];
    if (f < 0) return;
    const int it = ++lane_iter[b];
    const bool conv = !lane_unsat(unsat_mask, b, lw);
    if (!conv && it < max_iter) return;
    const int64_t j = f - first_frame;
    out_conv[j] = conv;
    out_iters[j] = conv ? it : max_iter;
    out_err[j] = !conv || ((lane_any[b >> lw] >> (b & ((1 << lw) - 1))) & 1u);
    const int64_t nf = atomicAdd(counts + 1, 1);
    if (nf < n_frames) {
        lane_frame[b] = first_frame + nf;
        lane_iter[b] = 0;
        refill[atomicAdd(counts, 1)] = (int32_t)b;
        atomicOr(fresh + (b >> lw), 1u << (b & ((1 << lw) - 1)));
    } else {
        lane_frame[b] = -1;
        active[b] = 0;
        atomicSub(n_active, 1);
    }
}

// New frames for the lanes in refill[0..counts[0]): Philox LLRs exactly as
// synth_llr_kernel (same (seed, snr_idx, frame) keying, all-zero word) into llr and
// L = clip(llr) + 0 (new_state).  Refill slots are strided over blockIdx.y, so the grid is
// small when (as in most sweeps) few or no lanes are refilled.
__device__ __forceinline__ void pool_refill_quad(int64_t b, int64_t qv, const int64_t *lane_frame, int64_t n, int lw,
                                                 uint64_t seed, uint32_t snr_idx, double sigma, double sigma2,
                                                 double clip, float *llr, float *L) {
    const int W = 1 << lw;
    const int64_t g = b >> lw, w = b & (W - 1);
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const uint64_t frame = (uint64_t)lane_frame[b];
    u32x4 ctr{(uint32_t)qv, (uint32_t)frame, (uint32_t)(frame >> 32), snr_idx & 0x7fffffffu};
    double nz[4];
    normals4(philox4x32_10(ctr, k0, k1), nz);
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int64_t v = qv * 4 + j;
        if (v >= n) break;
        const double r = 1.0 + sigma * nz[j];
        const float val = (float)(2.0 * r / sigma2);
        const int64_t idx = ((g * n + v) << lw) + w;
        llr[idx] = val;
        L[idx] = (float)clampT((double)val, clip) + 0.0f;
    }
}

__global__ void __launch_bounds__(kBlock) pool_refill_kernel(const int32_t *counts, const int32_t *refill,
                                                             const int64_t *lane_frame, int64_t n, int lw,
                                                             uint64_t seed, uint32_t snr_idx, double sigma,
                                                             double sigma2, double clip, float *llr, float *L) {
    const int64_t qv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (qv >= (n + 3) / 4) return;
    for (int slot = blockIdx.y; slot < counts[0]; slot += gridDim.y)
        pool_refill_quad(refill[slot], qv, lane_frame, n, lw, seed, snr_idx, sigma, sigma2, clip, llr, L);
}

__global__ void phi_array_kernel(const double *x, int64_t cnt, double eps, double clip, int prec, double *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    if (prec == 0)
        out[i] = (double)phi_fast((float)x[i], (float)eps, (float)clip);
    else
        out[i] = phi_ref(x[i], eps, clip);
}

}  // namespace qcl
