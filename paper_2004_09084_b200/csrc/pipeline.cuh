// pipeline.cuh -- TMA-pipelined layer update (sm_100a): bulk async copies + mbarriers.
//
// The direct kernel (layer_kernel) loads every operand into registers and computes in
// the same warps, so all resident warps of a wave load, then compute, then store in
// lockstep and HBM sits idle during the compute phase (ncu, profiles/README.md).  Here
// the two are decoupled:
//
//   warp 0 (producer)  walks this CTA's tiles; for tile t it issues one
//                      cp.async.bulk (UBLKCP) per contiguous run -- the posterior run of
//                      every circulant (one or two segments: the circulant wraps at z)
//                      and the edge-message run -- into stage t % S of a shared-memory
//                      ring, completing on the stage's "full" mbarrier;
//   warps 1..NC        wait "full", run the check update in place in shared memory, fence
//   (consumers)        the generic->async proxy and arrive on the stage's "empty" mbarrier;
//   warp 0             waits "empty" and bulk-stores the updated runs back
//                      (cp.async.bulk.global.shared::cta), then reuses the stage.
//
// A tile is (lane group g, slot s, checks k0..k0+KT-1) for all W lanes.  In shared memory
// tile element (edge j, check i, lane w) sits at j*KT*W + i*W + w for posteriors and
// (D + j)*KT*W + i*W + w for edge messages, so a consumer thread reads and writes V
// consecutive lanes with one vector LDS/STS and never touches global memory.
// Runs are multiples of W*sizeof(T) >= 16 bytes and 16-byte aligned (W >= 16/sizeof(T)).
#pragma once
#include <cstdint>

#include "kernels.cuh"

namespace qcl {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar,
                                          uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_store(void *gmem_dst, const void *smem_src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Warp-specialised pipeline: one producer warp + kConsumerWarps consumer warps per CTA.
// Every tile belongs to ONE consumer warp (tile i of the CTA -> warp i % C, stage
// i % S).  The consumer copies the stage into registers, releases it at once, computes
// and writes its results straight to global memory with coalesced vector stores, so
// the shared-memory ring only has to cover load latency (not compute) and the CTA can
// hold many consumer warps.
constexpr int kConsumerWarps = 11;
constexpr int kPipeThreads = 32 * (1 + kConsumerWarps);
constexpr int kMaxStages = 32;
constexpr int kRingBytes = 96 * 1024;

struct PipeArgs {
    SlotRange r;      // unit slot list, lanes
    void *L;
    void *R;
    const uint8_t *syn;
    int32_t KT;       // checks per tile
    int32_t kblocks;  // ceil(z / KT)
    int64_t tiles;    // G * nslots * kblocks
    int32_t stages;   // ring depth
    int32_t uniform;
    int32_t clip_r;   // clip can bind r (clip < Phi(eps)); otherwise the r clip is skipped
    double clip, eps;
};

struct TileGeom {
    int g, slot, k0, kt;
};
__device__ __forceinline__ TileGeom tile_geom(const PipeArgs &a, int64_t t64) {
    TileGeom tg;
    const uint32_t t = (uint32_t)t64;  // tiles < 2^31 (checked on the host)
    const uint32_t rest = t / (uint32_t)a.kblocks;
    const int kb = (int)(t - rest * (uint32_t)a.kblocks);
    const uint32_t gq = rest / (uint32_t)a.r.nslots;
    const int si = a.r.slot0 + (int)(rest - gq * (uint32_t)a.r.nslots);
    tg.g = (int)gq;
    tg.slot = a.r.slot_list ? a.r.slot_list[si] : si;
    tg.k0 = kb * a.KT;
    tg.kt = min(a.KT, a.r.z - tg.k0);
    return tg;
}

// Producer: lane j issues the bulk loads of circulant j of the tile (posterior run in one
// or two segments -- the circulant wraps at z -- and the edge-message run).
template <typename T>
__device__ __forceinline__ void tile_loads(const PipeArgs &a, const TileGeom &tg, T *stage, int D, uint64_t *bar,
                                           uint64_t pol_keep, uint64_t pol_stream) {
    const int lane = threadIdx.x & 31;
    const SlotInfo si = a.r.slots[tg.slot];
    const int W = 1 << a.r.lw, z = a.r.z;
    const int KTW = a.KT * W;
    const T *L = reinterpret_cast<const T *>(a.L);
    const T *R = reinterpret_cast<const T *>(a.R);
    for (int j = lane; j < si.degree; j += 32) {
        const EdgeInfo e = a.r.edges[si.edge_off + j];
        int p0 = tg.k0 + e.shift;
        p0 -= (p0 >= z) ? z : 0;
        const int len1 = min(tg.kt, z - p0);
        const uint32_t b1 = (uint32_t)len1 * W * sizeof(T);
        const uint32_t b2 = (uint32_t)(tg.kt - len1) * W * sizeof(T);
        const uint32_t br = (uint32_t)tg.kt * W * sizeof(T);
        // posteriors of multi-edge columns are re-read by later layers (keep them in L2);
        // degree-1 columns and edge messages are touched once per sweep (stream them)
        const uint64_t pl = e.reused ? pol_keep : pol_stream;
        T *ls = stage + (size_t)j * KTW;
        bulk_load(ls, L + (((int64_t)tg.g * a.r.n + e.var_base + p0) << a.r.lw), b1, bar, pl);
        if (b2) bulk_load(ls + (size_t)len1 * W, L + (((int64_t)tg.g * a.r.n + e.var_base) << a.r.lw), b2, bar, pl);
        bulk_load(stage + (size_t)(D + j) * KTW,
                  R + ((((int64_t)tg.g * a.r.E + si.edge_off + j) * z + tg.k0) << a.r.lw), br, bar, pol_stream);
    }
}

// Two CTAs per SM (22 consumer warps, <= 85 registers per thread) when the per-thread
// edge arrays are small (the degree-4 and degree-10/11 rows of the MET code in FP32),
// one otherwise.
template <typename T, int V, int D>
constexpr int pipe_min_blocks() {
    return (D * V * (int)sizeof(T) <= 64) ? 2 : 1;
}

template <typename T, int V, int D, bool HAS_SYN>
__global__ void __launch_bounds__(kPipeThreads, (pipe_min_blocks<T, V, D>())) layer_tma_kernel(PipeArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *empty = full + kMaxStages;
    T *stages = reinterpret_cast<T *>(smem_raw + 2 * kMaxStages * sizeof(uint64_t));
    const int W = 1 << a.r.lw;
    const int KTW = a.KT * W;
    const size_t stage_elems = (size_t)2 * D * KTW;
    const int S = a.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_local = a.tiles > blockIdx.x ? (a.tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer warp
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        for (int64_t i = 0; i < n_local; i++) {
            const int s = (int)(i % S);
            if (i >= S) mbar_wait(&empty[s], (uint32_t)((i / S) - 1) & 1);
            const TileGeom tg = tile_geom(a, blockIdx.x + i * gridDim.x);
            if (lane == 0) {
                const int d = a.r.slots[tg.slot].degree;
                mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * d * tg.kt * W * sizeof(T)));
            }
            __syncwarp();
            tile_loads<T>(a, tg, stages + (size_t)s * stage_elems, D, &full[s], pol_keep, pol_stream);
        }
        return;
    }

    // ---------------------------------------------------------------- consumer warps
    const int cw = warp - 1;
    const int lanes_v = W / V;
    const int items = KTW / (32 * V);  // items per thread per tile
    T *L = reinterpret_cast<T *>(a.L);
    T *R = reinterpret_cast<T *>(a.R);
    const T clip = (T)a.clip, eps = (T)a.eps;
    for (int64_t i = cw; i < n_local; i += kConsumerWarps) {
        const int s = (int)(i % S);
        const T *stage = stages + (size_t)s * stage_elems;
        const TileGeom tg = tile_geom(a, blockIdx.x + i * gridDim.x);
        const SlotInfo si = a.r.slots[tg.slot];
        const int d = si.degree;
        mbar_wait(&full[s], (uint32_t)(i / S) & 1);
        for (int sub = 0; sub < items; sub++) {
            const int item = sub * 32 + lane;
            const int ci = item / lanes_v;  // check within the tile
            const int w0 = (item - ci * lanes_v) * V;
            const bool live = ci < tg.kt;
            const int off = ci * W + w0;
            T q[D][V], ph[D][V];
            int par[V];
            if (HAS_SYN && live) {
                const uint8_t *sp =
                    a.syn + ((((int64_t)tg.g * a.r.S + tg.slot) * a.r.z + tg.k0 + ci) << a.r.lw) + w0;
#pragma unroll
                for (int v = 0; v < V; v++) par[v] = sp[v] & 1;
            } else {
#pragma unroll
                for (int v = 0; v < V; v++) par[v] = 0;
            }
            using VT = typename Vec<T, V>::type;
#pragma unroll
            for (int j = 0; j < D; j++) {
                if (j < d && live) {
                    T lv[V], rv[V];
                    *reinterpret_cast<VT *>(lv) = *reinterpret_cast<const VT *>(stage + (size_t)j * KTW + off);
                    *reinterpret_cast<VT *>(rv) = *reinterpret_cast<const VT *>(stage + (size_t)(D + j) * KTW + off);
#pragma unroll
                    for (int v = 0; v < V; v++) q[j][v] = clampT(lv[v] - rv[v], clip);
                } else {
#pragma unroll
                    for (int v = 0; v < V; v++) q[j][v] = (T)0;
                }
            }
            if (sub == items - 1) {
                // the whole tile is in registers: hand the stage back to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (!live) continue;
#pragma unroll
            for (int j = 0; j < D; j++) {
#pragma unroll
                for (int v = 0; v < V; v++) {
                    if (j < d) {
                        ph[j][v] = phi_absq<T>(q[j][v], eps);
                        par[v] ^= (q[j][v] < (T)0);
                    } else {
                        ph[j][v] = (T)0;
                    }
                }
            }
            others_in_place<T, V, D>(ph, d, a.uniform);
            const int k = tg.k0 + ci;
            const int64_t lbase = (int64_t)tg.g * a.r.n;
            const int64_t rbase = ((int64_t)tg.g * a.r.E + si.edge_off) * a.r.z + k;
#pragma unroll
            for (int j = 0; j < D; j++) {
                if (j < d) {
                    T rv[V], lv[V];
#pragma unroll
                    for (int v = 0; v < V; v++) {
                        T mag = phiT<T>(ph[j][v], eps, clip);
                        if (a.clip_r) mag = fmin(mag, clip);
                        rv[v] = ((q[j][v] < (T)0) ^ (par[v] != 0)) ? -mag : mag;
                        lv[v] = clampT(q[j][v] + rv[v], clip);
                    }
                    const EdgeInfo e = a.r.edges[si.edge_off + j];
                    int pos = k + e.shift;
                    pos -= (pos >= a.r.z) ? a.r.z : 0;
                    vstore<T, V>(R + ((rbase + (int64_t)j * a.r.z) << a.r.lw) + w0, rv);
                    vstore<T, V>(L + ((lbase + e.var_base + pos) << a.r.lw) + w0, lv);
                }
            }
        }
    }
}

}  // namespace qcl
