// flow.cuh -- persistent dataflow decode (sm_100a): every layer of every iteration in
// ONE launch, ordered by per-tile completion flags instead of kernel boundaries.
//
// Why.  The per-layer engines pay a launch ramp-up and a drain tail at each of the 30
// layer boundaries of a sweep (1500 per 50-iteration decode): a 2-row layer takes
// ~10 us although it moves 1.6 us worth of bytes (profiles/r01_launches_2iter_b64.csv).
// Layered decoding only orders a check after the checks that last wrote ITS variables
// (decoder.py:259-262 runs layer l+1 on the posteriors written by layer l), and in a
// QC code those writers are known statically: tile (slot s, checks k0..k0+kt) reads
// column c at offsets k + shift_s(c); the previous row p touching c wrote the same
// variables at offsets k + shift_s(c) - shift_p(c) (mod z).  So each tile waits for at
// most a few tiles of each previous writer, and the next layer starts as soon as the
// tiles it needs are stored instead of when the whole previous layer has drained.
//
// Work items are (iteration t, layer l, lane group g, slot s in l, k-block kb), in that
// order, claimed with one atomicAdd per tile.  A tile only waits for items claimed
// before it, so the kernel is deadlock free without co-residency: the smallest unfinished
// claimed item never waits (its dependencies are smaller, hence finished), and a CTA
// releases a tile's flag without waiting for anything else.  Lane groups interleave per
// layer, so with G groups a tile's dependencies were claimed at least (G-1) layer-groups
// earlier -- normally they are complete before it is claimed.
//
// Dependencies (flag[g][slot][kb] = iterations completed by that tile):
//   * RAW/WAR on posteriors: a tile waits for the previous writer's tiles that cover its
//     variables of every column (need t+1, or t if the previous writer is the same or a
//     later slot, i.e. in the previous iteration).  Each edge is a read-modify-write of
//     its variable by one check, so the RAW wait also orders every earlier read (WAR).
//   * edge messages R of (s, k) are only touched by (s, k) itself once per iteration;
//     every path of previous writers from (t-1, s, kb) to (t, s, kb) is a chain of such
//     waits, so the ordering is transitive (release/acquire at gpu scope).
//
// CTA roles (12 warps): warp 0 scheduler (claim, wait for dependencies, queue the tile
// header), warp 1 loader (bulk-load the tile's 2d runs into a ring stage), warps 2-3
// storers (alternate ring positions: bulk-store the updated stage, free it, wait for the
// writes, release the tile flag), warps 4..11 consumers (check update in shared memory,
// exactly the math of layer_tma_kernel).  The storers are what keep the scheme deadlock
// free: a scheduler blocked on a dependency never holds a finished tile back, because
// finished tiles are stored and released by other warps.
#pragma once
#include <cstdint>

#include "pipeline.cuh"

// Tile flags one per 128-byte line: neighbouring tiles' flags are written (release
// stores) and polled by different CTAs, and sharing a line costs ~7% at 64 codewords and
// ~30% at 16-32 (tools/flow_batches.sh; the polls of one line queue behind its writes).
#ifndef QCL_FLAG_STRIDE
#define QCL_FLAG_STRIDE 32  // ints between consecutive tile flags
#endif
#ifndef QCL_FLOW_STAGE_KB
#define QCL_FLOW_STAGE_KB 32
#endif
#ifndef QCL_FLOW_QUEUE
#define QCL_FLOW_QUEUE 1
#endif
#ifndef QCL_FLOW_ET_STOP
#define QCL_FLOW_ET_STOP 1  // fused ET: schedulers stop claiming once every frame converged
#endif
// role-warp waits: 0 = mbarrier try_wait with a suspend hint (wakes on barrier events);
// N > 0 = test_wait polling with an N ns back-off (tuning knobs, tools/flow_build_variants.sh)
#ifndef QCL_FLOW_STORER_SLEEP
#define QCL_FLOW_STORER_SLEEP 0
#endif
#ifndef QCL_FLOW_LOADER_SLEEP
#define QCL_FLOW_LOADER_SLEEP 0
#endif
#ifndef QCL_FLOW_CONSUMER_SLEEP
#define QCL_FLOW_CONSUMER_SLEEP 0
#endif
#define QCL_ROLE_WAIT(bar, par, ns) \
    do {                             \
        if (ns > 0)                  \
            mbar_wait_backoff(bar, par, ns); \
        else                         \
            mbar_wait_sleep(bar, par); \
    } while (0)

namespace qcl {

#ifndef QCL_FLOW_WIDE
#define QCL_FLOW_WIDE 0
#endif
// QCL_FLOW_WIDE = 0: two CTAs per SM, 8 consumer warps each; 1: one CTA per SM whose 16
// consumer warps share every tile (half the service time per tile, so half the time a
// claimed tile spends queued), with more storers and a deeper ring
constexpr int kFlowConsumers = QCL_FLOW_WIDE ? 16 : 8;  // consumer warps per CTA
#ifndef QCL_FLOW_STORERS
#define QCL_FLOW_STORERS (QCL_FLOW_WIDE ? 4 : 2)
#endif
// storer warps per CTA: storer k takes ring positions k, k + storers, ...; each must finish
// a stage's store, read-out wait and flag release (a GPU-scope fence) before its next one
constexpr int kFlowStorers = QCL_FLOW_STORERS;
constexpr int kFlowCtasPerSm = QCL_FLOW_WIDE ? 1 : 2;
constexpr int kFlowThreads = 32 * (kFlowConsumers + 2 + kFlowStorers);
constexpr int kFlowQueue = QCL_FLOW_QUEUE;         // scheduler -> loader header queue depth
constexpr int kFlowStageBytes = QCL_FLOW_STAGE_KB * 1024;  // one ring stage (2*D*KT*W floats)
constexpr int kFlowMaxStages = 6;
constexpr int kFlowHeadBytes = 512;                // mbarriers + stage headers + header queue

// Packed plan tables, copied into shared memory at kernel start (every producer/storer
// lookup is then an LDS, not a dependent L2 round trip).
//   slot: x = edge_off | degree << 16 | cls << 24,  y = kb_off (first tile flag in a group)
//   edge: x = col | reused << 15 | shift << 16,     y = prev_slot | wrap << 15 | delta << 16
// cls 0: d <= 4 (V 4), 1: d <= 8 (V 2), 2: d <= 12 (V 1); KT = 32 * consumers * V / W.
// prev_slot/wrap/delta: the previous writer of the column in cyclic schedule order and
// (shift - prev_shift) mod z; wrap = 1 when that writer runs in the previous iteration.
struct FlowHdr {  // stage header written by the producer, read by consumers and storers
    int32_t slot, g, k0, kt, d, cls, t, edge_off;
};

struct FlowArgs {
    const uint2 *slot_tab;   // [S]
    const uint2 *edge_tab;   // [E]
    const int2 *items;       // per item of one sweep: {slot | g << 16, kb}
    int32_t sweep_items;     // items per sweep of one group block
    uint32_t sweep_mul, sweep_shift;  // x / sweep_items == (umulhi(x, mul) + x) >> shift
    int32_t blk_items;       // items of this launch per group block (sweeps x sweep_items [+ tail])
    uint32_t blk_mul, blk_shift;      // x / blk_items, the same way
    int32_t item_end;        // items of this launch (group blocks x blk_items)
    int32_t tab_stride;      // item-table entries per group block (sweep_items [+ fused-ET tail])
    int32_t sweeps;          // sweeps of this launch; items past them are the fused-ET tail
    int32_t t_base;          // global sweep index of item 0 (flags count global sweeps)
    const int *t_dev;        // if set: t_base read from device memory (frame-pool sweep graphs)
    int *counter;            // claim counter of this launch (zeroed before it)
    int *flags;              // [G][nkb_total] iterations completed per tile
    int32_t nkb_total;
    void *L, *R;
    const uint8_t *syn;
    int64_t n;
    int32_t E, S, z, lw;
    int32_t stages;
    int32_t clip_r;
    const uint32_t *slot_mask;  // [S] bits 0-15: edge j's column is degree 1 (deferrable);
                                // bits 16-31: edge j is its column's last writer in a sweep
    const int *n_active;  // early termination: skip the launch once every frame converged
    const uint8_t *gactive;  // early termination: lane groups with an active frame (others skipped)
    int32_t defer_last;      // >= 0: degree-1 edges keep q in the L slot and no R until sweep defer_last
    const uint32_t *fresh;   // frame pool: [G] lanes that start a new frame this sweep (r_old = 0)
    int32_t fresh_t;         // sweep whose tiles treat every lane as fresh (a decode's first
                             // sweep: no zero fill of R before it), -1 none
    unsigned long long *stats;  // optional instrumentation (QCL_FLOW_STATS)
    double clip, eps;
    double mag_max;             // FP32 bound on |r| (LayerArgs::mag_max)
    float clip_f, mag_f;        // the same two, rounded to FP32 once on the host
    // fused early termination (flow_kernel<..., ETF = true>; W <= 8): every sweep of an ET
    // decode in this one launch, the per-sweep hard decision / syndrome check / freeze as
    // items of the same stream (see "Fused early termination" below)

    uint8_t *snap;           // [2][G][n] lane bits of the hard decision after sweep t (parity t & 1)
    uint8_t *fsign;          // [G][n] lane bits frozen at each lane's convergence
    int *cdone;              // [G] (x QCL_FLAG_STRIDE) check items completed, cumulative
    int *decided;            // [G] (x QCL_FLAG_STRIDE) sweeps whose ET decision is complete
    uint32_t *unsat;         // [2][G] (x QCL_FLAG_STRIDE) unsatisfied-lane masks, sweep parity
    uint32_t *amask;         // [G] lanes still active
    uint8_t *conv;           // [B] converged flags (decision)
    int64_t *iters;          // [B] iterations at convergence (decision)
    const uint32_t *synpack; // [S*z][G] packed target syndrome lane bits (nullptr: all zero)
    int32_t G;
    int32_t check_items;     // check items per lane group and sweep (slot ranges)
};

__host__ __device__ constexpr int flow_class_D(int cls) { return cls == 0 ? 4 : cls == 1 ? 8 : 12; }
// lanes per consumer thread by degree class (the tile is KT checks x W lanes shared by all
// consumer threads), and checks per tile: as many as the consumer threads cover, capped so
// that 2*D*KT*W floats fit one ring stage
__host__ __device__ constexpr int flow_class_V(int cls) {
    return kFlowConsumers >= 16 ? (cls == 0 ? 2 : 1) : (cls == 0 ? 4 : cls == 1 ? 2 : 1);
}
__host__ __device__ constexpr int flow_KT(int cls, int W) {
    return (kFlowConsumers * 32 * flow_class_V(cls) / W) < (kFlowStageBytes / (8 * flow_class_D(cls) * W))
               ? (kFlowConsumers * 32 * flow_class_V(cls) / W)
               : (kFlowStageBytes / (8 * flow_class_D(cls) * W));
}
// With the default 32 KB stage the stage cap never binds, so KT = 32 * consumers * V / W
// is a power of two and every tile index computation is a shift (the integer divisions
// they replace sat on the scheduler's per-item critical path).
__host__ __device__ constexpr int flow_ilog2(int x) { return x <= 1 ? 0 : 1 + flow_ilog2(x / 2); }
__host__ __device__ constexpr bool flow_kt_pow2() {
    return kFlowConsumers * 32 * flow_class_V(0) * 8 * flow_class_D(0) <= kFlowStageBytes &&
           kFlowConsumers * 32 * flow_class_V(1) * 8 * flow_class_D(1) <= kFlowStageBytes &&
           kFlowConsumers * 32 * flow_class_V(2) * 8 * flow_class_D(2) <= kFlowStageBytes;
}
// log2 KT (flow_kt_pow2() builds only)
__device__ __forceinline__ int flow_kt_log2(int cls, int lw) {
    return (cls == 0 ? flow_ilog2(kFlowConsumers * 32 * flow_class_V(0))
                     : cls == 1 ? flow_ilog2(kFlowConsumers * 32 * flow_class_V(1))
                                : flow_ilog2(kFlowConsumers * 32 * flow_class_V(2))) -
           lw;
}
// checks per tile on the device
__device__ __forceinline__ int flow_kt(int cls, int W, int lw) {
    if constexpr (flow_kt_pow2()) return 1 << flow_kt_log2(cls, lw);
    return flow_KT(cls, W);
}
// tile index of check offset k (k / KT)
__device__ __forceinline__ int flow_kb_of(int k, int cls, int W, int lw) {
    if constexpr (flow_kt_pow2()) return k >> flow_kt_log2(cls, lw);
    return k / flow_KT(cls, W);
}
// shared memory: head (mbarriers, headers) | slot table 8S | edge table 8E | last-writer
// bits 4S | consumer scratch 16 B | ring stages
__host__ __device__ constexpr size_t flow_table_end(int S, int E) {
    return ((kFlowHeadBytes + 8 * (size_t)(S + E) + 4 * (size_t)S + 16 + 127) / 128) * 128;
}
__host__ __device__ constexpr size_t flow_smem_bytes(int S, int E, int stages) {
    return flow_table_end(S, E) + (size_t)stages * kFlowStageBytes;
}

// Item n -> (sweep t relative to t_base, index into the item table), without divisions
// (n < 2^31, multipliers from flow_sweep_divisor).  Items run group block by group block
// (all sweeps of a launch for lane groups [b*GB, (b+1)*GB), then the next block), each
// block in (sweep, layer, group, slot, k-block) order.
__device__ __forceinline__ int flow_fastdiv(int x, uint32_t mul, uint32_t shift) {
    return (int)((__umulhi((uint32_t)x, mul) + (uint32_t)x) >> shift);
}
__device__ __forceinline__ int flow_item_map(const FlowArgs &a, int n, int &t) {
    const int b = flow_fastdiv(n, a.blk_mul, a.blk_shift);
    const int r = n - b * a.blk_items;
    t = flow_fastdiv(r, a.sweep_mul, a.sweep_shift);
    // the fused-ET tail (after the last sweep, t == sweeps) is stored after the sweep table
    return b * a.tab_stride + (t < a.sweeps ? 0 : a.sweep_items) + (r - t * a.sweep_items);
}
inline void flow_sweep_divisor(uint32_t d, uint32_t &mul, uint32_t &shift) {
    uint32_t l = 0;
    while ((1ull << l) < d) l++;
    mul = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    shift = l;
}

// QCL_FLOW_ACQUIRE: how a tile's dependency polls acquire the storers' releases.
//   0 (default): relaxed polls; the ordering rests on an sm_100 property, see spin_until;
//   1: ld.acquire.gpu on every flag load (a PTX-model synchronizes-with edge): +4.8% per
//      decode in bursts, +5.8% sustained (tools/flow_sustained.py, DESIGN 3.1);
//   2: relaxed polls, then one fence.acq_rel.gpu per resolved tile: +12%.
// QCL_FLOW_STATIC: item assignment.  0: dynamic claims (atomicAdd) everywhere; 1: static
// round-robin everywhere; 2 (default): static for the fused-ET kernel only.  Static
// kernels are launched cooperatively (co-residency is then guaranteed, which the static
// order needs for deadlock freedom).  No-ET decode: no difference (23.32 vs 23.34 ms
// sustained); fused-ET sweep 0.516 -> 0.493 ms (profiles/r02_ab_static.log).
#ifndef QCL_FLOW_STATIC
#define QCL_FLOW_STATIC 2
#endif
__host__ __device__ constexpr bool flow_static(bool etf) {
    return QCL_FLOW_STATIC == 1 || (QCL_FLOW_STATIC == 2 && etf);
}
#ifndef QCL_FLOW_ACQUIRE
#define QCL_FLOW_ACQUIRE 0
#endif
#if QCL_FLOW_ACQUIRE == 0 && defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 900 || __CUDA_ARCH__ >= 1100)
#error "relaxed flag polls are argued for sm_90..sm_10x bulk-copy semantics only; build with -DQCL_FLOW_ACQUIRE=1"
#endif
__device__ __forceinline__ int ld_flag(const int *p) {
    int v;
#if QCL_FLOW_ACQUIRE == 1
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#else
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#endif
    return v;
}
__device__ __forceinline__ void flow_acquire_fence() {
#if QCL_FLOW_ACQUIRE == 2
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Poll a tile flag.  Storer side (every variant): the tile's bulk writes complete
// (cp.async.bulk.wait_group 0: the writes are performed, i.e. in L2, the point of
// coherence for the async proxy) -> fence.proxy.async.global -> st.release.gpu of the
// flag.  Reader side:
//   QCL_FLOW_ACQUIRE = 1: the scheduler's ld.acquire.gpu that observes the flag
//   synchronizes with that release; its mbarrier arrive (release, CTA) -> the loader's
//   mbarrier wait (acquire, CTA) carries it to the loader (causality order is
//   transitive), whose fence.proxy.async.global orders its bulk reads after it.
//   QCL_FLOW_ACQUIRE = 0 (default): the same chain with a relaxed observing load.  The
//   PTX model gives no synchronizes-with edge for it; what makes it correct here is that
//   (a) the loader's bulk reads cannot be issued before the observation (they are data-
//   and control-dependent on the header the scheduler publishes after the poll returns),
//   and (b) cp.async.bulk reads are served by L2, where the released bytes already are
//   (no L1 copy can be stale for the async proxy).  That is an sm_90/sm_100 property,
//   hence the #error above for other architectures.  Measured cost of the formal
//   variant: +4.8% in bursts, +5.8% sustained; checked by tools/flow_stress.py (repeated
//   decodes bit-identical to the per-layer engine) and the bit-exact engine tests.
// abort (fused ET with static items): stop waiting once every frame has converged -- the
// tile waited for may belong to a CTA that has stopped; returns kSpinAborted then
constexpr int kSpinAborted = -(1 << 24);
__device__ __forceinline__ bool all_converged(const int *n_active) {
    return n_active && *(volatile const int *)n_active == 0;
}
__device__ __forceinline__ int spin_until(const int *flag, int need, const int *abort = nullptr) {
    if (ld_flag(flag) >= need) return 0;
    int polls = 1;
    while (ld_flag(flag) < need) {
        if (all_converged(abort)) return kSpinAborted;
        __nanosleep(64);
        polls++;
    }
    return polls;
}

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ bool spin_until_acquire(const int *flag, int need, const int *abort = nullptr) {
    while (ld_acquire_gpu(flag) < need) {
        if (all_converged(abort)) return false;
        __nanosleep(128);
    }
    return true;
}
__device__ __forceinline__ bool consumers_sync_or(bool p) {  // consumers_sync + OR of p
    uint32_t r;
    asm volatile(
        "{ .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, 1, %2, p;\n selp.u32 %0, 1, 0, q; }"
        : "=r"(r)
        : "r"((uint32_t)p), "n"(kFlowConsumers * 32)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ void red_release_max(int *p, int v) {
    asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Tile flag release.  With fused ET a tile of a converged group can be skipped (released at
// once) while an earlier-sweep tile of the same slot and k-block, resolved before the
// group converged, is still running: its later release must not lower the flag, or a
// waiter for the skipped tile's value would wait forever -- hence a max there.
__device__ __forceinline__ void flag_release(int *p, int v, bool monotonic) {
    if (monotonic)
        red_release_max(p, v);
    else
        st_release(p, v);
}
__device__ __forceinline__ void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acq_rel_add(int *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Bulk runs of one tile (LOAD: global -> stage, else stage -> global); lane j: edge j.
// RT: the edge-message type (float, or __half for 16-bit messages: the R run of edge j
// then fills the first half of its stage slot, so the stage layout does not change).
template <typename RT>
__device__ __forceinline__ void flow_runs(const FlowArgs &a, const FlowHdr &h, const uint2 *etab, int KT, int D,
                                          float *stage, uint64_t *bar, bool load, uint64_t pol_keep,
                                          uint64_t pol_stream) {
    const int lane = threadIdx.x & 31;
    const int W = 1 << a.lw, z = a.z;
    const int KTW = KT * W;
    float *Lg = reinterpret_cast<float *>(a.L) + (((size_t)h.g * a.n) << a.lw);
    RT *Rg = reinterpret_cast<RT *>(a.R) + ((((size_t)h.g * a.E + h.edge_off) * z + h.k0) << a.lw);
    for (int j = lane; j < h.d; j += 32) {
        const uint32_t ex = etab[h.edge_off + j].x;
        const int col = ex & 0x7fff, shift = ex >> 16;
        const bool reused = (ex >> 15) & 1;
        // degree-1 column under deferral (see flow_deferred): no R run moves, except the
        // final store of the last sweep
        const bool skip_r = !reused && a.defer_last >= 0 && (load || h.t != a.defer_last);
        int p0 = h.k0 + shift;
        p0 -= (p0 >= z) ? z : 0;
        const int len1 = min(h.kt, z - p0);
        const uint32_t b1 = (uint32_t)len1 * W * 4;
        const uint32_t b2 = (uint32_t)(h.kt - len1) * W * 4;
        const uint32_t br = (uint32_t)h.kt * W * (uint32_t)sizeof(RT);
        const uint64_t pl = reused ? pol_keep : pol_stream;
        const size_t vb = (size_t)col * z;
        float *lg1 = Lg + ((vb + p0) << a.lw);
        float *lg2 = Lg + (vb << a.lw);
        RT *rg = Rg + ((size_t)j * z << a.lw);
        float *ls = stage + (size_t)j * KTW;
        RT *rs = reinterpret_cast<RT *>(stage + (size_t)(D + j) * KTW);
        if (load) {
            bulk_load(ls, lg1, b1, bar, pl);
            if (b2) bulk_load(ls + (size_t)len1 * W, lg2, b2, bar, pl);
            if (!skip_r) bulk_load(rs, rg, br, bar, pol_stream);
        } else {
            bulk_store(lg1, ls, b1, pl);
            if (b2) bulk_store(lg2, ls + (size_t)len1 * W, b2, pl);
            if (!skip_r) bulk_store(rg, rs, br, pol_stream);
        }
    }
}

// Degree-1 deferral (bit-identical, fewer bytes).  A degree-1 column is touched by one
// check only, so between sweeps the only use of its posterior L and message R is the next
// sweep's q = clip(L - r) for that same edge.  Under deferral (the fused no-ET decode)
// the consumer computes that q right away, q' = clip(clip(q + r) - r) -- the very FP32
// operations the next sweep would do -- and leaves it in the L slot; no R moves.  The
// last sweep (t == defer_last) writes the true L = clip(q + r) and R = r, so the final
// state equals the undeferred one bit for bit.  Saves 8 of the 16 bytes per degree-1 edge
// and sweep (23% of the edges of the rate-0.1 code, ~19% of its DRAM traffic).
__device__ __forceinline__ uint32_t flow_deferred_mask(const FlowArgs &a, uint32_t smask) {
    return a.defer_last >= 0 ? (smask & 0xffffu) : 0u;  // bit j: edge j's column is degree 1
}

// V consecutive edge messages of one check <-> registers (FP32 or FP16 in the stage).
template <int V>
__device__ __forceinline__ void msg_load(const float *p, float (&r)[V]) {
    *reinterpret_cast<typename Vec<float, V>::type *>(r) = *reinterpret_cast<const typename Vec<float, V>::type *>(p);
}
template <int V>
__device__ __forceinline__ void msg_load(const __half *p, float (&r)[V]) {
    if constexpr (V == 1) {
        r[0] = __half2float(*p);
    } else {
        __half2 h[V / 2];
        if constexpr (V == 4)
            *reinterpret_cast<uint2 *>(h) = *reinterpret_cast<const uint2 *>(p);
        else
            *reinterpret_cast<uint32_t *>(h) = *reinterpret_cast<const uint32_t *>(p);
#pragma unroll
        for (int i = 0; i < V / 2; i++) {
            const float2 f = __half22float2(h[i]);
            r[2 * i] = f.x;
            r[2 * i + 1] = f.y;
        }
    }
}
template <int V>
__device__ __forceinline__ void msg_store(float *p, const float (&r)[V]) {
    *reinterpret_cast<typename Vec<float, V>::type *>(p) = *reinterpret_cast<const typename Vec<float, V>::type *>(r);
}
template <int V>
__device__ __forceinline__ void msg_store(__half *p, const float (&r)[V]) {  // r already FP16 values: exact
    if constexpr (V == 1) {
        *p = __float2half_rn(r[0]);
    } else {
        __half2 h[V / 2];
#pragma unroll
        for (int i = 0; i < V / 2; i++) h[i] = __floats2half2_rn(r[2 * i], r[2 * i + 1]);
        if constexpr (V == 4)
            *reinterpret_cast<uint2 *>(p) = *reinterpret_cast<const uint2 *>(h);
        else
            *reinterpret_cast<uint32_t *>(p) = *reinterpret_cast<const uint32_t *>(h);
    }
}
// consumer-warp barrier (named barrier 1): the FP16 generic path reuses R slots as FP32
// scratch, whose bytes overlap other threads' FP16 messages
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kFlowConsumers * 32) : "memory");
}

// ---- Fused early termination ---------------------------------------------------------
//
// decode_batch_arrays with early termination (decoder.py:295-305) checks every frame's hard
// decision against its syndrome after every sweep.  Here that check is part of the flow:
//  * snapshot: the consumers of a column's LAST writer in sweep t (slast bit) store the lane
//    bits of the new posteriors' signs as snap[t & 1][g][v] -- the hard decision after
//    sweep t, taken as it is produced (no pass over L);
//  * check items (per lane group, one per layer's slot range) of sweep t sit in the item
//    stream of sweep t + 1, after its first layers -- by then the tiles of sweep t are
//    stored, so a claimed check rarely waits.  A check item first reads the lanes already
//    known unsatisfied: if that covers every active lane (nearly always before
//    convergence) it has nothing to do; otherwise it waits until every tile of (g, t) is
//    stored (all the group's tile flags >= t + 1), XORs the snapshot bytes of each check
//    (^ target syndrome), stopping as soon as every active lane is unsatisfied, and ORs
//    the unsatisfied lanes into unsat[t & 1][g].  The last sweep's checks form a tail
//    after it;
//  * the check item that completes (g, t) (cdone) makes the decision: lanes newly satisfied
//    get converged / iterations = t + 1, their snapshot bits are frozen into fsign, and the
//    group stops being decoded once all its lanes converged (the rest of the launch skips
//    its items; once every frame converged the schedulers stop claiming).  Then it
//    releases decided[g] = t + 1.
//  * ordering: a tile with last-writer edges at sweep u >= 2 waits decided[g] >= u - 1
//    (the snapshot parity it overwrites has been read), and the checks of (g, t) wait
//    decided[g] >= t (decisions of a group stay in sweep order).  All waits point at items
//    claimed earlier, so the deadlock-freedom argument of the flow kernel holds.
// Outputs equal the per-sweep check: frames are independent, a converged lane's words are
// its snapshot at convergence, and lanes still active keep being updated as before.

// number of this warp's consumer lanes whose check lies inside the tile (those that did
// not return early): the shuffle mask of the snapshot combine
__device__ __forceinline__ unsigned flow_live_mask(int ct, int lv_log2, int kt) {
    const int live = (kt << lv_log2) - (ct & ~31);
    return live >= 32 ? 0xffffffffu : live <= 0 ? 0u : ((1u << live) - 1u);
}

// Snapshot of one edge's new posteriors x[0..V) (lanes w0..w0+V-1 of check ci): the W/V
// threads of the check OR their lane bits together; the one holding lane 0 stores the byte.
template <int V>
__device__ __forceinline__ void flow_snap(const FlowArgs &a, const FlowHdr &h, uint32_t ex, int ci, int w0,
                                          const float (&x)[V], unsigned mask) {
    uint32_t bits = 0;
#pragma unroll
    for (int v = 0; v < V; v++) bits |= (uint32_t)(x[v] < 0.0f) << (w0 + v);
    const int lv = (1 << a.lw) / V;
    for (int o = 1; o < lv; o <<= 1) bits |= __shfl_xor_sync(mask, bits, o);
    if (w0 == 0) {
        const int col = ex & 0x7fff, shift = ex >> 16;
        int pos = h.k0 + ci + shift;
        pos -= (pos >= a.z) ? a.z : 0;
        a.snap[((size_t)(h.t & 1) * a.G + h.g) * a.n + (size_t)col * a.z + pos] = (uint8_t)bits;
    }
}

// A check item (g, slots [h.slot, h.kt), sweep h.t), run by all consumer threads of the
// CTA; sc: 3 words of shared scratch.  See "Fused early termination" above.
__device__ __forceinline__ void flow_check(const FlowArgs &a, const FlowHdr &h, int ct, const uint2 *stab,
                                           const uint2 *etab, uint32_t *sc, bool abort_waits) {
    bool aborted = false;
    constexpr int kThreads = kFlowConsumers * 32;
    constexpr int kCk = 4;  // checks per thread in flight in a scan
    const int g = h.g, t = h.t, par = t & 1, z = a.z;
    uint32_t *unsat = a.unsat + ((size_t)par * a.G + g) * QCL_FLAG_STRIDE;
    uint32_t acc = 0;
    // lanes still to be decided: once every active lane is known unsatisfied (this
    // sweep's other check items, or this warp's own checks) no further check can change
    // the decision -- before convergence that is almost immediately, so most check items
    // scan a few checks, not z per slot
    const uint32_t need = __ldcg(a.amask + g);
    uint32_t known = __ldcg(unsat);
#ifndef QCL_FLOW_CHECK_EARLY
#define QCL_FLOW_CHECK_EARLY 1
#endif
    const bool scan = need && (!QCL_FLOW_CHECK_EARLY || (known & need) != need) && (!a.gactive || a.gactive[g]);
    if (scan) {
        // the snapshot of sweep t is complete once every tile of (g, t) is stored: all tile
        // flags of the group >= t + 1 (acquire; the barrier passes it to every thread)
        // relaxed polls, 8 in flight per thread, then one acquire fence per thread
        const int *fl = a.flags + (size_t)g * a.nkb_total * QCL_FLAG_STRIDE;
        for (int i0 = ct; i0 < a.nkb_total && !aborted; i0 += 8 * kThreads) {
            for (;;) {
                int v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int i = i0 + u * kThreads;
                    v[u] = i < a.nkb_total ? ld_flag(fl + (size_t)i * QCL_FLAG_STRIDE) : t + 1;
                }
                bool ok = true;
#pragma unroll
                for (int u = 0; u < 8; u++) ok &= v[u] >= t + 1;
                if (ok) break;
                if (abort_waits && all_converged(a.n_active)) {
                    aborted = true;
                    break;
                }
                __nanosleep(128);
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    // uniform: every consumer thread computed the same `scan`
    if (abort_waits) {
        if (consumers_sync_or(aborted)) return;  // every frame converged: nothing left to decide
    } else {
        consumers_sync();
    }
    const uint8_t *sg = a.snap + ((size_t)par * a.G + g) * a.n;
    // parity bits (lanes) of check k of slot s in this sweep's snapshot (^ target syndrome)
    auto check_bits = [&](int s, int k) {
        const uint32_t sx = stab[s].x;
        const int eo = sx & 0xffff, d = (sx >> 16) & 0xff;
        uint32_t b = a.synpack ? __ldg(a.synpack + ((size_t)s * z + k) * a.G + g) : 0u;
        for (int j = 0; j < d; j++) {
            const uint32_t ex = etab[eo + j].x;
            int pos = k + (int)(ex >> 16);
            pos -= (pos >= z) ? z : 0;
            b ^= __ldcg(sg + (size_t)(ex & 0x7fff) * z + pos);
        }
        return b;
    };
    // near convergence a codeword's few unsatisfied checks persist from sweep to sweep: the
    // check each lane failed last (hint[lane], id + 1) is tested first, which usually ends
    // the scan at once.  Which unsatisfied check is found does not matter for the decision.
    int *hint = a.cdone + (size_t)(4 * a.G + g) * QCL_FLAG_STRIDE;
    if (scan && ct < 32) {
        uint32_t hb = 0;
        if (ct < (1 << a.lw) && (((need & ~known) >> ct) & 1)) {
            const int id = __ldcg(hint + ct) - 1;
            if (id >= 0) hb = check_bits(id / z, id % z);
        }
        hb = __reduce_or_sync(0xffffffffu, hb);
        if (ct == 0) sc[2] = hb;
    }
    consumers_sync();
    if (scan) {
        acc = sc[2];
        known |= acc;
        bool done = (known & need) == need;
        for (int s = h.slot; s < h.kt && !done; s++) {  // h.kt: end of the slot range
            const uint32_t sx = stab[s].x;
            const int eo = sx & 0xffff, d = (sx >> 16) & 0xff;
            if ((z & 3) == 0) {
                // z a multiple of 4: each thread takes kCk quads of 4 consecutive checks; a
                // quad's bytes in one column are 4 consecutive bytes (mod z) = two aligned
                // words and a byte permute; all 2 d kCk word loads (L2 round trips) are issued
                // before the XORs
                for (int kw = (ct & ~31) * 4; kw < z; kw += kCk * kThreads * 4) {  // warp-uniform trips
                    const int k0 = kw + (ct & 31) * 4;
                    const uint32_t kn = (ct & 31) == 0 ? __ldcg(unsat) : 0u;  // other items' finds
                    uint32_t pb[kCk];
#pragma unroll
                    for (int u = 0; u < kCk; u++) {
                        const int k = k0 + u * kThreads * 4;
                        pb[u] = 0;
                        if (a.synpack && k < z) {
                            const uint32_t *sp = a.synpack + ((size_t)s * z + k) * a.G + g;
#pragma unroll
                            for (int i = 0; i < 4; i++) pb[u] |= __ldg(sp + (size_t)i * a.G) << (8 * i);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 12; j++) {
                        if (j < d) {
                            const uint32_t ex = etab[eo + j].x;
                            const uint32_t *colw = reinterpret_cast<const uint32_t *>(sg + (size_t)(ex & 0x7fff) * z);
                            const int sh = (int)(ex >> 16);
#pragma unroll
                            for (int u = 0; u < kCk; u++) {
                                const int k = k0 + u * kThreads * 4;
                                int pos = k + sh;
                                pos -= (pos >= z) ? z : 0;
                                const int w0 = pos >> 2, off = pos & 3;
                                const int w1 = (w0 + 1) * 4 == z ? 0 : w0 + 1;  // wraps at z
                                if (k < z)
                                    pb[u] ^= __byte_perm(__ldcg(colw + w0), __ldcg(colw + w1), 0x3210 + 0x1111 * off);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kCk; u++) {
                        const uint32_t x = pb[u];
                        const uint32_t lanes = (x | x >> 8 | x >> 16 | x >> 24) & 0xffu;
                        const uint32_t nw = lanes & need & ~known;
                        if (nw) {  // remember one failed check of the first new lane
                            const int l = __ffs(nw) - 1;
                            int i = 0;
                            while (!((x >> (8 * i + l)) & 1)) i++;
                            hint[l] = s * z + k0 + u * kThreads * 4 + i + 1;
                        }
                        acc |= lanes;
                    }
                    if (!QCL_FLOW_CHECK_EARLY) continue;
                    const uint32_t wacc = __reduce_or_sync(0xffffffffu, acc);
                    if ((ct & 31) == 0 && (wacc & need & ~known)) atomicOr(unsat, wacc);  // publish
                    known |= wacc | __shfl_sync(0xffffffffu, kn, 0);  // warp-uniform
                    if ((known & need) == need) {
                        done = true;
                        break;
                    }
                }
                continue;
            }
            // any z: four checks per thread in flight, all d x 4 byte loads issued before the XORs
            for (int kw = ct & ~31; kw < z; kw += kCk * kThreads) {  // warp-uniform trip count
                const int k0 = kw + (ct & 31);
                // the other check items of (g, t) publish what they find: re-read with the loads
                const uint32_t kn = (ct & 31) == 0 ? __ldcg(unsat) : 0u;
                uint32_t pb[kCk];
#pragma unroll
                for (int u = 0; u < kCk; u++) {
                    const int k = k0 + u * kThreads;
                    pb[u] = (a.synpack && k < z) ? __ldg(a.synpack + ((size_t)s * z + k) * a.G + g) : 0u;
                }
#pragma unroll
                for (int j = 0; j < 12; j++) {
                    if (j < d) {
                        const uint32_t ex = etab[eo + j].x;
                        const uint8_t *colp = sg + (size_t)(ex & 0x7fff) * z;
                        const int sh = (int)(ex >> 16);
#pragma unroll
                        for (int u = 0; u < kCk; u++) {
                            const int k = k0 + u * kThreads;
                            int pos = k + sh;
                            pos -= (pos >= z) ? z : 0;
                            if (k < z) pb[u] ^= __ldcg(colp + pos);  // L2: written by other CTAs
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kCk; u++) {
                    const uint32_t nw = pb[u] & need & ~known;
                    if (nw) hint[__ffs(nw) - 1] = s * z + k0 + u * kThreads + 1;
                    acc |= pb[u];
                }
                if (!QCL_FLOW_CHECK_EARLY) continue;
                const uint32_t wacc = __reduce_or_sync(0xffffffffu, acc);
                if ((ct & 31) == 0 && (wacc & need & ~known)) atomicOr(unsat, wacc);  // publish
                known |= wacc | __shfl_sync(0xffffffffu, kn, 0);  // warp-uniform
                if ((known & need) == need) {
                    done = true;
                    break;
                }
            }
        }
    }
    acc = __reduce_or_sync(0xffffffffu, acc);
    if (ct == 0) sc[0] = 0;
    consumers_sync();
    if ((ct & 31) == 0 && acc) atomicOr(&sc[0], acc);
    consumers_sync();
    if (ct == 0) {
        if (sc[0]) atomicOr(unsat, sc[0]);
        __threadfence();
        const int done = atom_acq_rel_add(a.cdone + (size_t)g * QCL_FLAG_STRIDE, 1) + 1;
        sc[1] = done == a.check_items * (t + 1);
    }
    consumers_sync();
    if (!sc[1]) return;  // uniform: read after the barrier
    // ---- decision for (g, t): this item completed the sweep's checks of the group
    if (ct == 0) {
        __threadfence();
        const uint32_t un = *(volatile uint32_t *)unsat;
        const uint32_t act = __ldcg(a.amask + g);  // L2: earlier decisions may have run on other SMs
        const uint32_t newm = act & ~un;
        sc[2] = newm;
        if (newm) {
            a.amask[g] = act & ~newm;
            for (uint32_t m = newm; m; m &= m - 1) {
                const int64_t b = ((int64_t)g << a.lw) + __ffs(m) - 1;
                a.conv[b] = 1;
                a.iters[b] = t + 1;
            }
            atomicSub(const_cast<int *>(a.n_active), __popc(newm));
            if (!(act & ~newm)) const_cast<uint8_t *>(a.gactive)[g] = 0;
        }
    }
    consumers_sync();
    const uint32_t newm = sc[2];
    if (newm) {  // freeze the newly converged lanes' words: fsign = snap where newm
        const uint8_t *sg = a.snap + ((size_t)par * a.G + g) * a.n;
        uint8_t *fg = a.fsign + (size_t)g * a.n;
        const uint32_t m4 = (newm & 0xffu) * 0x01010101u;
        const int64_t n16 = (a.n % 16 == 0) ? a.n / 16 : 0;  // 16-byte rows only when n is a multiple
        for (int64_t i = ct; i < n16; i += kThreads) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4 *>(sg) + i);
            uint4 f = __ldcg(reinterpret_cast<const uint4 *>(fg) + i);  // L2, as above
            f.x = (f.x & ~m4) | (x.x & m4);
            f.y = (f.y & ~m4) | (x.y & m4);
            f.z = (f.z & ~m4) | (x.z & m4);
            f.w = (f.w & ~m4) | (x.w & m4);
            reinterpret_cast<uint4 *>(fg)[i] = f;
        }
        for (int64_t v = n16 * 16 + ct; v < a.n; v += kThreads)
            fg[v] = (uint8_t)((__ldcg(fg + v) & ~newm) | (__ldcg(sg + v) & newm));
    }
    consumers_sync();
    if (ct == 0) {
        *(volatile uint32_t *)unsat = 0;  // reused by sweep t + 2, whose tiles wait for this release
        __threadfence();
        st_release(a.decided + (size_t)g * QCL_FLAG_STRIDE, t + 1);
    }
}

// One consumer thread: check (ci) of the tile for V lanes, in place in the stage.
// DF > 0: the slot's degree is DF; DMF >= 0: its deferral mask is DMF (compile-time
// specialisations of the common case -- every degree-4 row of the MET code has exactly one
// degree-1 column, its last edge -- which drop the per-edge degree/mask tests and the R
// stores the storer would skip anyway)
template <int V, int D, bool HAS_SYN, typename RT, bool ETF, int DF, int DMF>
__device__ __forceinline__ void flow_consume_body(const FlowArgs &a, const FlowHdr &h, float *stage, int ct,
                                                  const uint2 *etab, uint32_t smask) {
    const int d = DF > 0 ? DF : h.d;
    const uint32_t lastm = smask >> 16;
    const int W = 1 << a.lw;
    const int KT = flow_kt(h.cls, W, a.lw);
    const int KTW = KT * W;
    const int lv_log2 = a.lw - flow_ilog2(V);  // W / V lanes per check (W >= V)
    const int ci = ct >> lv_log2;
    const int w0 = (ct - (ci << lv_log2)) * V;
    if (ci >= h.kt) return;
    const int off = ci * W + w0;
    const float clip = a.clip_f;
    constexpr bool H = sizeof(RT) == 2;
    using VT = typename Vec<float, V>::type;
    float q[D][V], ph[D][V];
    int par[V];
    const uint32_t dmask = DMF >= 0 ? (uint32_t)DMF : flow_deferred_mask(a, smask);
    const bool last = h.t == a.defer_last;
    const uint32_t fresh_lanes = h.t == a.fresh_t ? 0xffffffffu : a.fresh ? a.fresh[h.g] : 0u;
    if (HAS_SYN) {
        const uint8_t *sp = a.syn + ((((int64_t)h.g * a.S + h.slot) * a.z + h.k0 + ci) << a.lw) + w0;
#pragma unroll
        for (int v = 0; v < V; v++) par[v] = sp[v] & 1;
    } else {
#pragma unroll
        for (int v = 0; v < V; v++) par[v] = 0;
    }
#pragma unroll
    for (int j = 0; j < D; j++) {
        if (j < d) {
            float lv[V], rv[V];
            *reinterpret_cast<VT *>(lv) = *reinterpret_cast<const VT *>(stage + (size_t)j * KTW + off);
            if ((dmask >> j) & 1) {  // the L slot already holds q
#pragma unroll
                for (int v = 0; v < V; v++) q[j][v] = lv[v];
            } else {
                msg_load<V>(reinterpret_cast<const RT *>(stage + (size_t)(D + j) * KTW) + off, rv);
                if (fresh_lanes) {  // frame pool: lanes that just took a new frame have r_old = 0
#pragma unroll
                    for (int v = 0; v < V; v++)
                        if ((fresh_lanes >> (w0 + v)) & 1) rv[v] = 0.0f;
                }
#pragma unroll
                for (int v = 0; v < V; v++) q[j][v] = clampT(lv[v] - rv[v], clip);
            }
        } else {
#pragma unroll
            for (int v = 0; v < V; v++) q[j][v] = 0.0f;
        }
    }
    if (D == 4 && d == 4) {
        uint32_t sb[V];
#pragma unroll
        for (int v = 0; v < V; v++) sb[v] = (uint32_t)par[v] << 31;
        check_update_f32_d4<V, H>(reinterpret_cast<float(&)[4][V]>(q), reinterpret_cast<float(&)[4][V]>(ph), sb,
                                  a.mag_f, clip);
    } else {
        check_update_f32<V, D, H>(q, ph, par, d, a.mag_f, clip);
    }
    if (ETF && lastm) {  // fused ET: hard-decision snapshot of the columns this slot writes last
        const unsigned mask = flow_live_mask(ct, lv_log2, h.kt);
#pragma unroll
        for (int j = 0; j < D; j++)
            if (j < d && ((lastm >> j) & 1)) flow_snap<V>(a, h, etab[h.edge_off + j].x, ci, w0, q[j], mask);
    }
#pragma unroll
    for (int j = 0; j < D; j++) {
        if (j < d) {
            const bool deferred = (dmask >> j) & 1;
            if (deferred && !last) {  // next sweep's q for a deferred degree-1 edge
#pragma unroll
                for (int v = 0; v < V; v++) q[j][v] = clampT(q[j][v] - ph[j][v], clip);
            }
            // a deferred edge's R run is stored only in the last sweep (flow_runs)
            if (DMF < 0 || !deferred || last)
                msg_store<V>(reinterpret_cast<RT *>(stage + (size_t)(D + j) * KTW) + off, ph[j]);
            *reinterpret_cast<VT *>(stage + (size_t)j * KTW + off) = *reinterpret_cast<VT *>(q[j]);
        }
    }
}

template <int V, int D, bool HAS_SYN, typename RT, bool ETF>
__device__ __forceinline__ void flow_consume(const FlowArgs &a, const FlowHdr &h, float *stage, int ct,
                                             const uint2 *etab, uint32_t smask) {
    if constexpr (D == 4) {
        const uint32_t dm = flow_deferred_mask(a, smask);
        if (h.d == 4 && dm == 8u) return flow_consume_body<V, D, HAS_SYN, RT, ETF, 4, 8>(a, h, stage, ct, etab, smask);
        if (h.d == 4 && dm == 0u) return flow_consume_body<V, D, HAS_SYN, RT, ETF, 4, 0>(a, h, stage, ct, etab, smask);
    }
    flow_consume_body<V, D, HAS_SYN, RT, ETF, 0, -1>(a, h, stage, ct, etab, smask);
}

// Degree classes 1 and 2 (rows of degree 5..12): the sum/difference update with the
// exclusive prefix (S, D) pairs stashed in the tile's own shared-memory slots of each edge
// (free once the edge's L and R are in registers) instead of registers, so the 80-register
// budget of two resident CTAs per SM holds without spills.  Same arithmetic, in the same
// order, as check_update_f32.  With FP16 messages the FP32 stash overlaps other threads'
// FP16 R values, so all consumers read their inputs before the first stash write and keep
// the new messages in registers until every thread has read its stash back.
template <int V, int D, bool HAS_SYN, typename RT, bool ETF>
__device__ __forceinline__ void flow_consume_gen(const FlowArgs &a, const FlowHdr &h, float *stage, int ct,
                                                 const uint2 *etab, uint32_t smask) {
    const uint32_t lastm = smask >> 16;
    constexpr bool H = sizeof(RT) == 2;
    const int W = 1 << a.lw;
    const int KT = flow_kt(h.cls, W, a.lw);
    const int KTW = KT * W;
    const int lv_log2 = a.lw - flow_ilog2(V);  // W / V lanes per check (W >= V)
    const int ci = ct >> lv_log2;
    const int w0 = (ct - (ci << lv_log2)) * V;
    const bool act = ci < h.kt;
    if (!H && !act) return;
    const int off = ci * W + w0;
    const float clip = a.clip_f, mag_max = a.mag_f;
    using VT = typename Vec<float, V>::type;
    float q[D][V], t[D][V];
    int par[V];
    const uint32_t fresh_lanes = h.t == a.fresh_t ? 0xffffffffu : a.fresh ? a.fresh[h.g] : 0u;
    const uint32_t dmask = flow_deferred_mask(a, smask);
    const bool last = h.t == a.defer_last;
    if (HAS_SYN && act) {
        const uint8_t *sp = a.syn + ((((int64_t)h.g * a.S + h.slot) * a.z + h.k0 + ci) << a.lw) + w0;
#pragma unroll
        for (int v = 0; v < V; v++) par[v] = sp[v] & 1;
    } else {
#pragma unroll
        for (int v = 0; v < V; v++) par[v] = 0;
    }
#pragma unroll
    for (int j = 0; j < D; j++) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            q[j][v] = 0.0f;
            t[j][v] = 0.0f;
        }
        if (j < h.d && act) {
            float lv[V], rv[V];
            *reinterpret_cast<VT *>(lv) = *reinterpret_cast<const VT *>(stage + (size_t)j * KTW + off);
            msg_load<V>(reinterpret_cast<const RT *>(stage + (size_t)(D + j) * KTW) + off, rv);
            const bool dj = (dmask >> j) & 1;  // the L slot already holds q
#pragma unroll
            for (int v = 0; v < V; v++) {
                if ((fresh_lanes >> (w0 + v)) & 1) rv[v] = 0.0f;  // frame pool: new frame, r_old = 0
                q[j][v] = dj ? lv[v] : clampT(lv[v] - rv[v], clip);
                t[j][v] = sd_t(q[j][v]);
                par[v] ^= (q[j][v] < 0.0f);
            }
        }
    }
    if (H) consumers_sync();
    if (act) {
        // exclusive prefix (S, D) pairs -> the edge's L / R slots
        float ps[V], pd[V];
#pragma unroll
        for (int v = 0; v < V; v++) {
            ps[v] = 1.0f;
            pd[v] = 0.0f;
        }
#pragma unroll
        for (int j = 0; j < D; j++) {
            if (j < h.d) {
                *reinterpret_cast<VT *>(stage + (size_t)j * KTW + off) = *reinterpret_cast<VT *>(ps);
                *reinterpret_cast<VT *>(stage + (size_t)(D + j) * KTW + off) = *reinterpret_cast<VT *>(pd);
#pragma unroll
                for (int v = 0; v < V; v++) {
                    const float ns = fmaf(t[j][v], pd[v], ps[v]);
                    pd[v] = fmaf(t[j][v], ps[v], pd[v]);
                    ps[v] = ns;
                }
            }
        }
        float ss[V], sd[V];
#pragma unroll
        for (int v = 0; v < V; v++) {
            ss[v] = 1.0f;
            sd[v] = 0.0f;
        }
#pragma unroll
        for (int j = D - 1; j >= 0; j--) {
            if (j < h.d) {
                float xs[V], xd[V], rr[V], ll[V], lsn[V];
                *reinterpret_cast<VT *>(xs) = *reinterpret_cast<const VT *>(stage + (size_t)j * KTW + off);
                *reinterpret_cast<VT *>(xd) = *reinterpret_cast<const VT *>(stage + (size_t)(D + j) * KTW + off);
#pragma unroll
                for (int v = 0; v < V; v++) {
                    const float S = fmaf(xs[v], ss[v], xd[v] * sd[v]), Dv = fmaf(xs[v], sd[v], xd[v] * ss[v]);
                    const float mag = msg_round<H>(sd_mag(S, Dv, mag_max));
                    rr[v] = ((q[j][v] < 0.0f) ^ (par[v] != 0)) ? -mag : mag;
                    ll[v] = clampT(q[j][v] + rr[v], clip);
                    lsn[v] = ll[v];  // the new posterior (its sign is the hard decision)
                    if (((dmask >> j) & 1) && !last) ll[v] = clampT(ll[v] - rr[v], clip);  // deferred: next q
                    const float ns = fmaf(t[j][v], sd[v], ss[v]);
                    sd[v] = fmaf(t[j][v], ss[v], sd[v]);
                    ss[v] = ns;
                }
                if (ETF && ((lastm >> j) & 1))  // fused ET snapshot of the new posteriors
                    flow_snap<V>(a, h, etab[h.edge_off + j].x, ci, w0, lsn, flow_live_mask(ct, lv_log2, h.kt));
                if (H) {  // the R slot may still hold another thread's stash: r waits in q[j]
#pragma unroll
                    for (int v = 0; v < V; v++) q[j][v] = rr[v];
                } else {
                    *reinterpret_cast<VT *>(stage + (size_t)(D + j) * KTW + off) = *reinterpret_cast<VT *>(rr);
                }
                *reinterpret_cast<VT *>(stage + (size_t)j * KTW + off) = *reinterpret_cast<VT *>(ll);
            }
        }
    }
    if (H) {
        consumers_sync();
        if (act) {
#pragma unroll
            for (int j = 0; j < D; j++)
                if (j < h.d) msg_store<V>(reinterpret_cast<RT *>(stage + (size_t)(D + j) * KTW) + off, q[j]);
        }
    }
}

#define FLOW_TICK(k)                          \
    if (prof) {                               \
        const long long c_ = clock64();       \
        acc[k] += c_ - tc;                    \
        tc = c_;                              \
    }

// ETF: fused early termination (a separate instantiation, so that the no-ET kernel carries
// none of its code: the snapshot path alone cost the no-ET decode ~4% through register
// allocation)
template <bool HAS_SYN, bool PROF, typename RT = float, bool ETF = false>
__global__ void __launch_bounds__(kFlowThreads, kFlowCtasPerSm) flow_kernel(FlowArgs a) {
    if (a.n_active && *(volatile const int *)a.n_active == 0) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);  // loader -> consumers (+tx)
    uint64_t *done = full + kFlowMaxStages;                    // consumers -> storers
    uint64_t *empty = done + kFlowMaxStages;                   // storers -> loader
    uint64_t *ready = empty + kFlowMaxStages;                  // scheduler -> loader (queue)
    uint64_t *qfree = ready + kFlowQueue;                      // loader -> scheduler (queue)
    FlowHdr *hdr = reinterpret_cast<FlowHdr *>(smem_raw + 256);
    FlowHdr *hq = hdr + kFlowMaxStages;
    uint2 *stab = reinterpret_cast<uint2 *>(smem_raw + kFlowHeadBytes);
    uint2 *etab = stab + a.S;
    uint32_t *slt = reinterpret_cast<uint32_t *>(etab + a.E);  // slot masks (last-writer bits with ETF only)
    uint32_t *scratch = slt + a.S;                              // check items (consumers)
    float *stages = reinterpret_cast<float *>(smem_raw + flow_table_end(a.S, a.E));
    constexpr size_t kStageElems = kFlowStageBytes / 4;
    const int S = a.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = 1 << a.lw;

    for (int i = threadIdx.x; i < a.S; i += blockDim.x) stab[i] = a.slot_tab[i];
    for (int i = threadIdx.x; i < a.E; i += blockDim.x) etab[i] = a.edge_tab[i];
    for (int i = threadIdx.x; i < a.S; i += blockDim.x) slt[i] = a.slot_mask[i] & (ETF ? 0xffffffffu : 0xffffu);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], kFlowConsumers);
            mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < kFlowQueue; q++) {
            mbar_init(&ready[q], 1);
            mbar_init(&qfree[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr bool prof = PROF;  // instrumented build (QCL_FLOW_STATS): phase cycle counters
    long long acc[4] = {0, 0, 0, 0}, tc = 0;

    if (warp == 0) {
        // ----------------------------------------------------------------- scheduler
        // claims run two items ahead and the item record one ahead, so neither L2 round
        // trip is on the tile's critical path.  Holding claimed items is deadlock free:
        // they are larger than the item in hand.  Resolved headers go to the loader warp
        // through a small queue, so dependency polling overlaps the bulk-copy issue.
        const int t_base = a.t_dev ? *(volatile const int *)a.t_dev : a.t_base;
        int n2 = 0;
        // stop: every frame converged (fused ET) -- the items already claimed (the one in
        // hand and the prefetched one) are still processed, nothing new is claimed
        bool stop = false;
        // static round-robin items (flow_static<ETF>: launched cooperatively, so every
        // CTA is co-resident and a CTA's items wait only on earlier items of running CTAs)
        constexpr bool kStatic = flow_static(ETF);
        if (kStatic) n2 = blockIdx.x;
        else if (lane == 0) n2 = atomicAdd(a.counter, 1);
        auto next_claim = [&]() {
            if constexpr (kStatic) {
                const int n = n2;
                if (n < a.item_end) n2 = stop ? a.item_end : n + (int)gridDim.x;
                return n;
            } else {
                const int n = __shfl_sync(0xffffffffu, n2, 0);
                if (n < a.item_end && lane == 0) n2 = stop ? a.item_end : atomicAdd(a.counter, 1);
                return n;
            }
        };
        auto record = [&](int n) {
            int t;
            return __ldg(a.items + flow_item_map(a, n, t));
        };
        int n1 = next_claim();
        int2 r1 = make_int2(0, 0);
        if (n1 < a.item_end) r1 = record(n1);
        int sentinels = 0;
        unsigned long long n_waited = 0, n_polls = 0, n_tiles = 0;
        // fused ET: lane (g & 31) caches the largest decided[g] it has observed (monotonic),
        // so the snapshot-reuse gate costs an L2 round trip once per group and sweep, not
        // once per tile
        int dec_tag = -1, dec_val = 0;
        // lane j < d: the flags of the previous writer of edge j's column covering this
        // tile's offsets (kb in [lo, lo + nlo) and, past the wrap at z, [0, nfl - nlo))
        auto flag_plan = [&](const FlowHdr &h, const int *&fl, int &need, int &lo, int &nlo, int &nfl) {
            nfl = 0;
            if (lane >= h.d) return;
            const uint32_t dy = etab[h.edge_off + lane].y;
            need = h.t + 1 - (int)((dy >> 15) & 1);
            if (need <= 0) return;
            const uint2 pst = stab[dy & 0x7fff];
            const int pcls = pst.x >> 24;
            fl = a.flags + ((size_t)h.g * a.nkb_total + pst.y) * QCL_FLAG_STRIDE;
            int a0 = h.k0 + (int)(dy >> 16);
            a0 -= (a0 >= a.z) ? a.z : 0;
            const int b = a0 + h.kt - 1;
            lo = flow_kb_of(a0, pcls, W, a.lw);
            nlo = flow_kb_of(min(b, a.z - 1), pcls, W, a.lw) - lo + 1;
            nfl = nlo + (b >= a.z ? flow_kb_of(b - a.z, pcls, W, a.lw) + 1 : 0);
        };
        auto resolve = [&](int item, int2 e) {
            FlowHdr h;
            int t_rel;
            flow_item_map(a, item, t_rel);
            h.t = t_base + t_rel;
            h.slot = e.x & 0xffff;
            h.g = e.x >> 16;
            const uint2 st = stab[h.slot];
            h.edge_off = st.x & 0xffff;
            h.d = (st.x >> 16) & 0xff;
            h.cls = st.x >> 24;
            if (e.y < 0) {  // fused-ET check item: every check of slots [slot, -1 - e.y) after the
                h.k0 = -1;  // PREVIOUS sweep (the items of sweep t's checks sit in sweep t + 1's
                h.kt = -1 - e.y;  // stream, so their tiles are long stored when they are claimed)
                h.t -= 1;
                return h;
            }
            const int KT = flow_kt(h.cls, W, a.lw);
            h.k0 = e.y * KT;
            h.kt = min(KT, a.z - h.k0);
            return h;
        };
        for (int it = 0, q = 0, ph = 0;; it++) {
            if (prof) tc = clock64();
            if (it >= kFlowQueue) mbar_wait_sleep(&qfree[q], ph ^ 1);
            FLOW_TICK(0);
            const int item = n1;
            const int2 e = r1;
            if (item >= a.item_end) {
                // one end marker per storer warp, at consecutive ring positions
                if (lane == 0) {
                    hq[q].kt = -1;
                    mbar_arrive(&ready[q]);
                }
                if (++sentinels == kFlowStorers) break;
            } else {
                n1 = next_claim();
                if (n1 < a.item_end) r1 = record(n1);
                FLOW_TICK(1);
                const FlowHdr h = resolve(item, e);
                if (h.k0 < 0 && h.t < 0) {  // the first sweep's check items (of sweep -1): nothing
                    __syncwarp();
                    goto next_item;
                }
                if (h.k0 >= 0 && a.gactive && !a.gactive[h.g]) {
                    // every frame of this lane group has converged: its outputs are frozen,
                    // so the tile is not updated -- only released for the group's later tiles
                    __syncwarp();
                    if (lane == 0) {
                        flag_release(a.flags + ((size_t)h.g * a.nkb_total + stab[h.slot].y + e.y) * QCL_FLAG_STRIDE, h.t + 1,
                                     ETF);
                    }
                    if (QCL_FLOW_ET_STOP && ETF) {
                        int none = 0;
                        if (lane == 0) none = *(volatile const int *)a.n_active == 0;
                        stop = stop || __shfl_sync(0xffffffffu, none, 0);
                    }
                    goto next_item;
                }
                // wait for the previous writers of every column of this tile: all covering
                // flags of an edge are loaded together (one round trip), only stale ones polled
                int polls = 0;
                // static items: a wait may point at a tile whose CTA stopped after every frame
                // converged -- abort it then (nothing observable is left to compute)
                const int *abort = (kStatic && ETF && QCL_FLOW_ET_STOP) ? a.n_active : nullptr;
                if (h.k0 < 0) {
                    // check item (g, slot, t): every tile of (g, t) stored, decisions in order
                    if (lane == 0 && h.t >= 1 && !spin_until_acquire(a.decided + (size_t)h.g * QCL_FLAG_STRIDE, h.t, abort))
                        polls = kSpinAborted;
                    __syncwarp();
                } else {
                    if (ETF && (slt[h.slot] >> 16) && h.t >= 2) {  // snapshot parity reuse
                        const int owner = h.g & 31;
                        const bool cached = __shfl_sync(0xffffffffu, dec_tag == h.g && dec_val >= h.t - 1, owner);
                        if (!cached && lane == owner) {
                            const int *dp = a.decided + (size_t)h.g * QCL_FLAG_STRIDE;
                            polls += spin_until(dp, h.t - 1, abort);
                            dec_tag = h.g;
                            dec_val = h.t - 1;
                        }
                    }
                    const int *fl = nullptr;
                    int need = 0, lo = 0, nlo = 0, nfl = 0, fv[4];
                    flag_plan(h, fl, need, lo, nlo, nfl);
#pragma unroll
                    for (int m = 0; m < 4; m++)
                        if (m < nfl) fv[m] = ld_flag(fl + (m < nlo ? lo + m : m - nlo) * QCL_FLAG_STRIDE);
#pragma unroll
                    for (int m = 0; m < 4; m++)
                        if (m < nfl && fv[m] < need) polls += spin_until(fl + (m < nlo ? lo + m : m - nlo) * QCL_FLAG_STRIDE, need, abort);
                    for (int m = 4; m < nfl; m++) polls += spin_until(fl + (m < nlo ? lo + m : m - nlo) * QCL_FLAG_STRIDE, need, abort);
                }
                if (abort && __any_sync(0xffffffffu, polls < 0)) {
                    stop = true;  // every frame converged: this item and the rest are dropped
                    goto next_item;
                }
                flow_acquire_fence();
                FLOW_TICK(2);
                if (prof) {
                    polls = __reduce_add_sync(0xffffffffu, polls);
                    n_waited += polls != 0;
                    n_polls += polls;
                    n_tiles++;
                }
                __syncwarp();
                if (lane == 0) {
                    hq[q] = h;
                    mbar_arrive(&ready[q]);  // release: the loader's bulk reads follow these polls
                }
                FLOW_TICK(3);
            }
            if (++q == kFlowQueue) {
                q = 0;
                ph ^= 1;
            }
            continue;
        next_item:
            it--;  // nothing was queued: this queue slot is still free
        }
        if (prof && lane == 0) {
            for (int k = 0; k < 4; k++) atomicAdd(a.stats + 3 + k, (unsigned long long)acc[k]);
            atomicAdd(a.stats, n_waited);
            atomicAdd(a.stats + 1, n_polls);
            atomicAdd(a.stats + 2, n_tiles);
        }
        return;
    }

    if (warp == 1) {
        // -------------------------------------------------------------------- loader
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        int sentinels = 0;
        const bool lprof = PROF;
        for (int it = 0, s = 0, ph = 0, q = 0, qph = 0;; it++) {
            if (lprof) tc = clock64();
            QCL_ROLE_WAIT(&ready[q], qph, QCL_FLOW_LOADER_SLEEP);
            if (lprof) { const long long c_ = clock64(); acc[0] += c_ - tc; tc = c_; }
            const FlowHdr h = hq[q];
            __syncwarp();
            if (lane == 0) mbar_arrive(&qfree[q]);
            if (++q == kFlowQueue) {
                q = 0;
                qph ^= 1;
            }
            if (it >= S) QCL_ROLE_WAIT(&empty[s], ph ^ 1, QCL_FLOW_LOADER_SLEEP);
            if (lprof) { const long long c_ = clock64(); acc[1] += c_ - tc; tc = c_; }
            if (h.kt < 0) {
                if (lane == 0) {
                    hdr[s].kt = -1;
                    mbar_arrive(&full[s]);
                }
                if (++sentinels == kFlowStorers) break;
            } else if (h.k0 < 0) {  // fused-ET check item: no bulk data, the consumers read L2
                if (lane == 0) {
                    hdr[s] = h;
                    mbar_arrive(&full[s]);
                }
                __syncwarp();
            } else {
                fence_proxy_async_global();  // observed flags -> ordered before the bulk (async proxy) reads
                const int KT = flow_kt(h.cls, W, a.lw);
                // runs moved: d L runs, plus the R runs of edges not under degree-1 deferral
                const uint32_t nr = (uint32_t)h.d - __popc(flow_deferred_mask(a, slt[h.slot]));
                if (lane == 0) {
                    hdr[s] = h;
                    mbar_arrive_expect_tx(&full[s], ((uint32_t)h.d * 4 + nr * (uint32_t)sizeof(RT)) * (uint32_t)(h.kt * W));
                }
                __syncwarp();
                flow_runs<RT>(a, h, etab, KT, flow_class_D(h.cls), stages + (size_t)s * kStageElems, &full[s], true,
                          pol_keep, pol_stream);
                __syncwarp();
                if (lprof) acc[2] += clock64() - tc;
            }
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
        if (lprof && lane == 0) {
            atomicAdd(a.stats + 7, (unsigned long long)acc[1]);
            atomicAdd(a.stats + 8, (unsigned long long)acc[2]);
            atomicAdd(a.stats + 15, (unsigned long long)acc[0]);
        }
        return;
    }

    if (warp <= 1 + kFlowStorers) {
        // ------------------------------------------------------------------- storers
        // storer k takes ring positions k, k + kFlowStorers, ...: one warp's wait for its
        // writes to complete overlaps the other's stores
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        const bool sprof = PROF && warp == 2;
        for (int it = warp - 2;; it += kFlowStorers) {
            const int s = it % S;
            if (sprof) tc = clock64();
            QCL_ROLE_WAIT(&done[s], (it / S) & 1, QCL_FLOW_STORER_SLEEP);
            if (sprof) { const long long c_ = clock64(); acc[0] += c_ - tc; tc = c_; }
            const FlowHdr h = hdr[s];
            if (h.kt < 0) break;
            if (h.k0 < 0) {  // check item: nothing to store
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                continue;
            }
            const int KT = flow_kt(h.cls, W, a.lw);
            flow_runs<RT>(a, h, etab, KT, flow_class_D(h.cls), stages + (size_t)s * kStageElems, nullptr, false,
                      pol_keep, pol_stream);
            bulk_commit();
            if (sprof) { const long long c_ = clock64(); acc[1] += c_ - tc; tc = c_; }
            bulk_wait_read_all();  // the stage may be refilled once its bytes are read out
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (sprof) { const long long c_ = clock64(); acc[2] += c_ - tc; tc = c_; }
            bulk_wait_all();  // this lane's writes are performed ...
            fence_proxy_async_global();
            __syncwarp();
            if (lane == 0) {  // ... before the tile is released to its dependents
                flag_release(a.flags + ((size_t)h.g * a.nkb_total + stab[h.slot].y + flow_kb_of(h.k0, h.cls, W, a.lw)) * QCL_FLAG_STRIDE,
                             h.t + 1, ETF);
            }
            if (sprof) acc[3] += clock64() - tc;
        }
        if (sprof && lane == 0)
            for (int k = 0; k < 4; k++) atomicAdd(a.stats + 11 + k, (unsigned long long)acc[k]);
        return;
    }

    // ---------------------------------------------------------------------- consumers
    const int ct = threadIdx.x - 32 * (2 + kFlowStorers);
    const bool cprof = PROF && warp == 2 + kFlowStorers;
    int sentinels = 0;
    for (int s = 0, ph = 0;;) {
        if (cprof) tc = clock64();
        QCL_ROLE_WAIT(&full[s], ph, QCL_FLOW_CONSUMER_SLEEP);
        if (cprof) { const long long c_ = clock64(); acc[0] += c_ - tc; tc = c_; }
        const FlowHdr h = hdr[s];
        if (h.kt < 0) {
            if (lane == 0) mbar_arrive(&done[s]);
            if (++sentinels == kFlowStorers) break;
        } else {
            float *stage = stages + (size_t)s * kStageElems;
            if (ETF && h.k0 < 0) {
                if constexpr (ETF) flow_check(a, h, ct, stab, etab, scratch, flow_static(ETF) && QCL_FLOW_ET_STOP);
            } else if (h.cls == 0) {
                flow_consume<flow_class_V(0), 4, HAS_SYN, RT, ETF>(a, h, stage, ct, etab, slt[h.slot]);
            } else if (h.cls == 1) {
                flow_consume_gen<flow_class_V(1), 8, HAS_SYN, RT, ETF>(a, h, stage, ct, etab, slt[h.slot]);
            } else {
                flow_consume_gen<flow_class_V(2), 12, HAS_SYN, RT, ETF>(a, h, stage, ct, etab, slt[h.slot]);
            }
            fence_proxy_async_smem();  // this thread's STS -> visible to the bulk-store engine
            __syncwarp();
            if (lane == 0) mbar_arrive(&done[s]);
            if (cprof) acc[1] += clock64() - tc;
        }
        if (++s == S) {
            s = 0;
            ph ^= 1;
        }
    }
    if (cprof && lane == 0)
        for (int k = 0; k < 2; k++) atomicAdd(a.stats + 9 + k, (unsigned long long)acc[k]);
}
#undef FLOW_TICK

}  // namespace qcl
