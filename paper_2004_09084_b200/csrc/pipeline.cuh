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
// Same wait with a suspend-time hint: the warp sleeps in the barrier unit until the phase
// completes (or the hint elapses) instead of re-issuing try_wait, so idle roles (flow
// engine) leave their issue slots to the consumer warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000)
        : "memory");
}
// Polling wait with a fixed back-off (no barrier-event wake-ups): for role warps whose
// reaction latency is not on the critical path (QCL_FLOW_*_SLEEP tuning in flow.cuh).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity, unsigned ns) {
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
    }
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

// All consumer warps of a CTA work on the same tile: tile = (lane group g, slot s, checks
// k0..k0+KT-1) for all W lanes with KT = 32*kConsumerWarps*V/W, one (check, V-lane)
// item per consumer thread.  The stage is updated in place; the producer writes it
// back with bulk stores before reusing it.  Every consumer waits for every phase of
// every stage in order, so mbarrier parities cannot alias.
constexpr int kMaxStages = 4;

struct PipeArgs {
    SlotRange r;      // unit slot list, lanes
    void *L;
    void *R;
    const uint8_t *syn;
    int32_t KT;       // checks per tile
    int32_t kblocks;  // ceil(z / KT)
    int64_t tiles;    // G * nslots * kblocks  (< 2^31)
    int32_t stages;   // ring depth (<= kMaxStages)
    int32_t uniform;
    int32_t clip_r;
    const int *n_active;  // early termination: skip the launch once every frame converged
    double clip, eps;
    double mag_max;       // FP32 bound on |r| (LayerArgs::mag_max)
};

struct TileGeom {
    int g, slot, k0, kt;
};
__device__ __forceinline__ TileGeom tile_geom(const PipeArgs &a, int64_t t64) {
    TileGeom tg;
    const uint32_t t = (uint32_t)t64;
    const uint32_t rest = t / (uint32_t)a.kblocks;
    const int kb = (int)(t - rest * (uint32_t)a.kblocks);
    const uint32_t gq = rest / (uint32_t)a.r.nslots;
    const int si = a.r.slot0 + (int)(rest - gq * (uint32_t)a.r.nslots);
    tg.g = a.r.g0 + (int)gq;
    tg.slot = a.r.slot_list ? a.r.slot_list[si] : si;
    tg.k0 = kb * a.KT;
    tg.kt = min(a.KT, a.r.z - tg.k0);
    return tg;
}

// Issue (LOAD) or write back (!LOAD) every run of a tile.  Lane j handles circulant j:
// posterior run in one or two segments (the circulant wraps at z), edge-message run.
template <typename T, bool LOAD>
__device__ __forceinline__ void tile_runs(const PipeArgs &a, const TileGeom &tg, T *stage, int D, uint64_t *bar,
                                          uint64_t pol_keep, uint64_t pol_stream) {
    const int lane = threadIdx.x & 31;
    const SlotInfo si = a.r.slots[tg.slot];
    const int W = 1 << a.r.lw, z = a.r.z;
    const int KTW = a.KT * W;
    T *Lg = reinterpret_cast<T *>(a.L) + (((size_t)tg.g * a.r.n) << a.r.lw);
    T *Rg = reinterpret_cast<T *>(a.R) + ((((size_t)tg.g * a.r.E + si.edge_off) * z + tg.k0) << a.r.lw);
    for (int j = lane; j < si.degree; j += 32) {
        const EdgeInfo e = a.r.edges[si.edge_off + j];
        int p0 = tg.k0 + e.shift;
        p0 -= (p0 >= z) ? z : 0;
        const int len1 = min(tg.kt, z - p0);
        const uint32_t b1 = (uint32_t)len1 * W * sizeof(T);
        const uint32_t b2 = (uint32_t)(tg.kt - len1) * W * sizeof(T);
        const uint32_t br = (uint32_t)tg.kt * W * sizeof(T);
        // posteriors of multi-edge columns are re-read by later layers (keep in L2);
        // degree-1 columns and edge messages are touched once per sweep (stream)
        const uint64_t pl = e.reused ? pol_keep : pol_stream;
        T *lg1 = Lg + ((size_t)(e.var_base + p0) << a.r.lw);
        T *lg2 = Lg + ((size_t)e.var_base << a.r.lw);
        T *rg = Rg + ((size_t)j * z << a.r.lw);
        T *ls = stage + (size_t)j * KTW;
        T *rs = stage + (size_t)(D + j) * KTW;
        if (LOAD) {
            bulk_load(ls, lg1, b1, bar, pl);
            if (b2) bulk_load(ls + (size_t)len1 * W, lg2, b2, bar, pl);
            bulk_load(rs, rg, br, bar, pol_stream);
        } else {
            bulk_store(lg1, ls, b1, pl);
            if (b2) bulk_store(lg2, ls + (size_t)len1 * W, b2, pl);
            bulk_store(rg, rs, br, pol_stream);
        }
    }
}

template <typename T, int V, int D, int C>
constexpr int pipe_min_blocks() {
    return (D * V * (int)sizeof(T) <= 64) ? (C <= 4 ? 3 : 2) : 1;
}

// C consumer warps per CTA (template), a.stages ring stages (runtime).
template <typename T, int V, int D, bool HAS_SYN, int C>
__global__ void __launch_bounds__(32 * (C + 1), (pipe_min_blocks<T, V, D, C>())) layer_tma_kernel(PipeArgs a) {
    constexpr int kConsumerWarps = C;
    pdl_launch_dependents();  // see layer_kernel
    pdl_wait();
    if (a.n_active && *(volatile const int *)a.n_active == 0) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *empty = full + kMaxStages;
    const int kStages = a.stages;
    T *stages = reinterpret_cast<T *>(smem_raw + 128);
    const int W = 1 << a.r.lw;
    const int KTW = a.KT * W;
    const size_t stage_elems = (size_t)2 * D * KTW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------------------------------------------------------- producer
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        int it = 0;
        for (int64_t t = blockIdx.x; t < a.tiles; t += gridDim.x, it++) {
            const int s = it % kStages;
            T *stage = stages + (size_t)s * stage_elems;
            if (it >= kStages) {
                // the stage holds tile t - S*grid: wait for its update, write it back
                mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
                const TileGeom old = tile_geom(a, t - (int64_t)kStages * gridDim.x);
                tile_runs<T, false>(a, old, stage, D, nullptr, pol_keep, pol_stream);
                bulk_commit();
                bulk_wait_read_all();  // the stage's smem may be overwritten after this
                __syncwarp();
            }
            const TileGeom tg = tile_geom(a, t);
            if (lane == 0) {
                const int d = a.r.slots[tg.slot].degree;
                mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * d * tg.kt * W * sizeof(T)));
            }
            __syncwarp();
            tile_runs<T, true>(a, tg, stage, D, &full[s], pol_keep, pol_stream);
        }
        // drain: write back the last (up to S) tiles
        for (int k = max(0, it - kStages); k < it; k++) {
            const int s = k % kStages;
            mbar_wait(&empty[s], (k / kStages) & 1);
            const TileGeom old = tile_geom(a, blockIdx.x + (int64_t)k * gridDim.x);
            tile_runs<T, false>(a, old, stages + (size_t)s * stage_elems, D, nullptr, pol_keep, pol_stream);
        }
        bulk_commit();
        bulk_wait_all();
        return;
    }

    // -------------------------------------------------------------------- consumers
    const int ct = threadIdx.x - 32;
    const int lanes_v = W / V;
    const int ci = ct / lanes_v;  // check within the tile
    const int w0 = (ct - ci * lanes_v) * V;
    const int off = ci * W + w0;
    LayerArgs la;  // numeric parameters for check_update
    la.uniform = a.uniform;
    la.clip_r = a.clip_r;
    la.clip = a.clip;
    la.eps = a.eps;
    la.mag_max = a.mag_max;
    const T clip = (T)a.clip;
    using VT = typename Vec<T, V>::type;
    int it = 0;
    for (int64_t t = blockIdx.x; t < a.tiles; t += gridDim.x, it++) {
        const int s = it % kStages;
        T *stage = stages + (size_t)s * stage_elems;
        const TileGeom tg = tile_geom(a, t);
        const int d = a.r.slots[tg.slot].degree;
        mbar_wait(&full[s], (it / kStages) & 1);
        if (ci < tg.kt) {
            T q[D][V], ph[D][V];
            int par[V];
            if (HAS_SYN) {
                const uint8_t *sp =
                    a.syn + ((((int64_t)tg.g * a.r.S + tg.slot) * a.r.z + tg.k0 + ci) << a.r.lw) + w0;
#pragma unroll
                for (int v = 0; v < V; v++) par[v] = sp[v] & 1;
            } else {
#pragma unroll
                for (int v = 0; v < V; v++) par[v] = 0;
            }
#pragma unroll
            for (int j = 0; j < D; j++) {
                if (j < d) {
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
            check_update<V, D>(q, ph, par, d, la);
#pragma unroll
            for (int j = 0; j < D; j++) {
                if (j < d) {
                    *reinterpret_cast<VT *>(stage + (size_t)(D + j) * KTW + off) = *reinterpret_cast<VT *>(ph[j]);
                    *reinterpret_cast<VT *>(stage + (size_t)j * KTW + off) = *reinterpret_cast<VT *>(q[j]);
                }
            }
        }
        fence_proxy_async_smem();  // this thread's STS -> visible to the bulk-store engine
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

}  // namespace qcl
