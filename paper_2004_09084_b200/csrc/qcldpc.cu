// qcldpc.cu -- plan, device state, launch sequencing and the C ABI (include/qcldpc_b200.h).
//
// The reference decoder (decoder.py:108-312) is a numpy loop: for t in iterations,
// for layer in schedule, one vectorised _layer_update_core.  Here the same loop nest
// runs on the device: the packed H_compact1 table lives in HBM for the life of the
// plan, every layer is one kernel launch over all checks of all merged rows of that
// layer for all codewords of the batch, and one sweep (all layers) is captured once
// into a CUDA graph that is replayed per iteration, so the host issues one graph
// launch per iteration instead of ~30 kernel launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/qcldpc_b200.h"
#include "kernels.cuh"
#include "pipeline.cuh"
#include "flow.cuh"
#include "hostio.h"

using namespace qcl;

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(QCL_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Every entry point runs on its plan's device and gives the calling thread its current
// device back on return (callers such as torch rely on it).
struct DeviceScope {
    int prev = -1;
    bool ok = false;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = prev == dev || cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope &) = delete;
    DeviceScope &operator=(const DeviceScope &) = delete;
};
#define DEVICE_SCOPE(dev)                                                           \
    DeviceScope dscope_(dev);                                                       \
    if (!dscope_.ok) return fail(QCL_ECUDA, "cudaSetDevice(%d) failed", (int)(dev))

// FP32 bound on |r|: Phi(eps) (the reference clamps `others` to >= eps, decoder.py:104),
// and the clip where it binds (decoder.py:244-245).
static double mag_bound(double clip, double eps) { return std::min(clip, log1p(2.0 / expm1(eps))); }

struct qcl_plan {
    int device = 0;
    int z = 0, n_cols = 0, S = 0, n_layers = 0, E = 0;
    int64_t n = 0, m = 0;
    int max_degree = 0;
    std::vector<int32_t> layer_start;  // [n_layers + 1] slot ranges
    std::vector<int> layer_dmax, layer_uniform;
    // launch units: the rows of a merged layer are independent, so a ragged layer is
    // split by degree class and each class gets the kernel variant sized for it
    struct Unit {
        int layer, list_off, count, dmax;
    };
    std::vector<Unit> units;
    std::vector<int> layer_unit0;  // [n_layers + 1]
    int32_t *slot_list = nullptr;  // device: concatenated unit slot ids
    std::vector<int32_t> h_slot_list;
    std::vector<SlotInfo> h_slots;
    SlotInfo *slots = nullptr;  // device H_compact1: per slot
    EdgeInfo *edges = nullptr;  // device H_compact1: per circulant
    uint2 *fedge_tab = nullptr;  // device, flow engine: packed circulant + previous-writer table
    uint32_t *fslast = nullptr;  // device, flow engine: per slot, bits 0-15: edge j's column is degree 1,
                                 // bits 16-31: edge j writes its column last in a sweep (flow.cuh)
    int32_t *funtouched = nullptr;  // device: columns no row touches (their decisions never change)
    int n_untouched = 0;
    bool flow_ok = false;        // the code fits the flow engine's packed tables
    std::vector<int32_t> h_edge_shift, h_edge_col;
    std::mutex cache_mu;
    std::vector<qcl_state *> cache;  // idle states reused by qcl_decode
};

constexpr int kSideStreams = 8;

struct qcl_state {
    qcl_plan *plan = nullptr;
    cudaStream_t side[kSideStreams] = {};
    cudaEvent_t fork = nullptr, join[kSideStreams] = {};
    int64_t B = 0, Bp = 0;
    int prec = QCL_PREC_FP32, lw = 0, W = 1, G = 1;
    int api_prec = QCL_PREC_FP32;  // as created; prec is the posterior type (FP32 for MSG16)
    bool msg16 = false;            // FP16 edge messages (QCL_PREC_FP32_MSG16, flow engine only)
    size_t esz = 4, resz = 4;      // posterior / edge-message element sizes
    cudaStream_t stream = nullptr;
    void *llr = nullptr, *L = nullptr, *R = nullptr;
    uint8_t *syn = nullptr;  // lanes layout, valid if has_syn
    bool has_syn = false;
    uint8_t *words = nullptr, *conv = nullptr, *active = nullptr, *take = nullptr;
    uint8_t *gactive = nullptr;  // [G] lane groups with an active frame (early termination)
    uint32_t *unsat = nullptr;    // [G] lane bit masks of unsatisfied codewords
    uint32_t *signs = nullptr;    // [G][n] packed hard decisions
    uint32_t *synpack = nullptr;  // [G][S][z] packed target syndrome (valid if has_syn)
    int64_t *iters = nullptr;
    int *n_active = nullptr, *h_n_active = nullptr;  // device / pinned host
    uint8_t *truths = nullptr;
    bool truths_valid = false;  // the last synthetic fill was encode mode (else all-zero words)
    void *staging = nullptr;
    size_t staging_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void *staging2 = nullptr;  // syndrome staging (async path: LLR staging may still be in flight)
    size_t staging2_bytes = 0;
    int engine = 4;  // flow engine where eligible, else the TMA per-layer kernels
    // per-sweep CUDA graph, rebuilt when clip/eps/syndrome presence change
    cudaGraphExec_t sweep_exec = nullptr;
    double g_clip = -1, g_eps = -1;
    bool g_syn = false, g_et = false;  // graph key; g_et: layer kernels skip once all converged
    cudaEvent_t ev_flag[2] = {};        // early-termination flag copies, one iteration behind
    // whole-decode graph and its key
    cudaGraphExec_t decode_exec = nullptr;
    double d_clip = -1, d_eps = -1;
    bool d_syn = false, d_et = false;
    int d_iters = -1, d_engine = -1;
    int64_t d_launches_layer = 0, d_launches_all = 0;
    int *h_flag = nullptr;              // pinned [2]
    int64_t launches_layer = 0, launches_all = 0, sweep_launches = 0;
    bool profiling = false;
    float layer_ms = 0;
    // flow engine (engine 4): tiling, item list, tile flags and claim counters
    uint2 *fslot_tab = nullptr;
    int2 *fitems = nullptr;
    int *fflags = nullptr, *fcounters = nullptr;
    unsigned long long *fstats = nullptr;  // QCL_FLOW_STATS=1: dependency-wait counters
    int64_t f_sweep_items = 0;  // items per sweep of one group block
    int32_t f_nblk = 1;         // group blocks (flow.cuh flow_item_map)
    int32_t f_nkb_total = 0, f_counter_cap = 0, f_grid = 0, f_stages = 3;
    bool flow_decode = false;  // this decode runs on the flow engine
    bool fused_et = false;     // this decode's early termination runs inside the flow launch
    // fused early termination (flow.cuh): item list with check items, snapshot buffers
    int2 *fitems_et = nullptr;
    int64_t f_sweep_items_et = 0;  // per sweep of one group block (its table adds a tail)
    int32_t f_check_items = 0;     // check items per lane group and sweep
    uint8_t *fsnap = nullptr;   // [2][G][n]
    uint8_t *fsign = nullptr;   // [G][n]
    int *fet = nullptr;         // cdone | decided | unsat[2] | hint, each [G] x QCL_FLAG_STRIDE
    uint32_t *famask = nullptr; // [G]
    // frame pool (qcl_state_decode_pool): per lane frame index / iterations, refill list
    bool pool_active = false;
    int64_t *pframe = nullptr;     // [Bp] frame decoded by the lane, -1 idle
    int32_t *piter = nullptr;      // [Bp] iterations of the lane's current frame
    uint32_t *pfresh = nullptr;    // [G] lanes that start a new frame in the next sweep
    uint32_t *plane_any = nullptr; // [G] lanes whose hard decision has a set bit
    int32_t *prefill = nullptr;    // [Bp] lanes to refill this sweep
    int32_t *pcount = nullptr;     // [0] refills this sweep, [1] frames handed out
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> sweep_events;
    // persistent per-layer engine (W <= 2 lanes): unit table of one sweep, barrier counter
    PersistUnit *punits = nullptr;
    unsigned *pbar = nullptr;
    int p_nu = 0, p_grid = 0, p_maxd = 4;
    double p_clip = -1, p_eps = -1;
    bool p_syn = false;
    bool persist_decode = false;  // this decode runs on the persistent per-layer engine
    HostRing ring;  // pinned chunks of the pageable-memory copy pipelines (hostio.h)
};

// ----------------------------------------------------------------------------- dispatch

static int env_int(const char *name, int dflt);

// Per-layer kernels are launched with programmatic dependent launch (QCL_PDL, default on):
// a layer's grid is scheduled while the previous layer drains and waits in
// griddepcontrol.wait (kernels.cuh) before touching state, which hides most of the
// launch gap of the ~1500 dependent launches of a per-layer decode (the small-batch and
// single-codeword path, BASELINE configs[1]).
template <typename Arg>
static void launch_pdl(void (*kern)(Arg), dim3 grid, dim3 block, size_t smem, cudaStream_t s, const Arg &a) {
    static const bool on = env_int("QCL_PDL", 1) != 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = on ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename T, int V, int DMAX>
static void launch_layer_t(const LayerArgs &a, dim3 grid, cudaStream_t s, bool syn) {
    if (syn)
        launch_pdl(layer_kernel<T, V, DMAX, true>, grid, dim3(kBlock), 0, s, a);
    else
        launch_pdl(layer_kernel<T, V, DMAX, false>, grid, dim3(kBlock), 0, s, a);
}

// Only the (V, DMAX) pairs vec_width() can select are instantiated: wide vectors are
// used for low-degree layers only, so their per-thread arrays never spill.
template <typename T, int V>
static void launch_layer_v(const LayerArgs &a, int dmax, dim3 grid, cudaStream_t s, bool syn) {
    constexpr int kMaxD = V == 1 ? 32 : (sizeof(T) == 4 ? 16 / V : 4);
    if (dmax <= 4)
        launch_layer_t<T, V, 4>(a, grid, s, syn);
    else if (dmax <= 8 && kMaxD >= 8)
        launch_layer_t<T, V, (kMaxD >= 8 ? 8 : 4)>(a, grid, s, syn);
    else if (dmax <= 12 && kMaxD >= 12)
        launch_layer_t<T, V, (kMaxD >= 12 ? 12 : 4)>(a, grid, s, syn);
    else if (dmax <= 16 && kMaxD >= 16)
        launch_layer_t<T, V, (kMaxD >= 16 ? 16 : 4)>(a, grid, s, syn);
    else if (kMaxD >= 32)
        launch_layer_t<T, V, (kMaxD >= 32 ? 32 : 4)>(a, grid, s, syn);
}

// Lanes per thread: wide vectors for the degree-4 layers that dominate the MET code,
// narrower ones for high-degree rows so the per-thread edge arrays stay in registers
// (fp32: DMAX 4/V 4 -> 64 regs, DMAX 8/V 2 -> 75, DMAX 12/V 1 -> 74; see ptxas -v).
static int vec_width(const qcl_state *st, int dmax) {
    int v;
    if (st->prec == QCL_PREC_FP32)
        v = dmax <= 4 ? 4 : (dmax <= 8 ? 2 : 1);
    else
        v = dmax <= 4 ? 2 : 1;
    return std::min(st->W, v);
}

static SlotRange slot_range(const qcl_state *st, int slot0, int nslots, int V, const int32_t *list = nullptr) {
    const qcl_plan *p = st->plan;
    SlotRange r;
    r.slot_list = list;
    r.slots = p->slots;
    r.edges = p->edges;
    r.n = p->n;
    r.E = p->E;
    r.S = p->S;
    r.z = p->z;
    r.slot0 = slot0;
    r.nslots = nslots;
    r.bps = (int)cdiv((int64_t)p->z * (st->W / V), kBlock);
    r.lw = st->lw;
    r.g0 = 0;
    return r;
}

// ------------------------------------------------------------ TMA-pipelined units
static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <typename T, int V, int D, bool SYN, int C>
static void launch_tma_tc(const PipeArgs &a, cudaStream_t stream) {
    auto kern = layer_tma_kernel<T, V, D, SYN, C>;
    const size_t smem = 128 + (size_t)a.stages * 2 * D * C * 32 * V * sizeof(T);
    static int configured_smem = -1, sms = 0;
    if (configured_smem < (int)smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured_smem = (int)smem;
    }
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int blocks_per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, 32 * (C + 1), smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    const int64_t grid = std::min<int64_t>(a.tiles, (int64_t)sms * blocks_per_sm);
    launch_pdl(kern, dim3((unsigned)grid), dim3(32 * (C + 1)), smem, stream, a);
}

// consumer warps per CTA: 8 by default (QCL_PIPE_WARPS=4 selects the 4-warp variant)
static int pipe_warps() {
    static int w = env_int("QCL_PIPE_WARPS", 8) == 4 ? 4 : 8;
    return w;
}

template <typename T, int V, int D, bool SYN>
static void launch_tma_t(const PipeArgs &a, cudaStream_t stream) {
    if (pipe_warps() == 4)
        launch_tma_tc<T, V, D, SYN, 4>(a, stream);
    else
        launch_tma_tc<T, V, D, SYN, 8>(a, stream);
}

template <typename T, int V, int D>
static void launch_tma_d(const PipeArgs &a, cudaStream_t stream, bool syn) {
    if (syn)
        launch_tma_t<T, V, D, true>(a, stream);
    else
        launch_tma_t<T, V, D, false>(a, stream);
}

template <typename T>
static void launch_tma(const PipeArgs &a, int V, int dmax, cudaStream_t stream, bool syn) {
    if (V == 4 && sizeof(T) == 4)
        launch_tma_d<T, (sizeof(T) == 4 ? 4 : 2), 4>(a, stream, syn);
    else if (V == 2 && sizeof(T) == 4)
        launch_tma_d<T, 2, 8>(a, stream, syn);
    else if (V == 2)
        launch_tma_d<T, 2, 4>(a, stream, syn);
    else if (dmax <= 4)
        launch_tma_d<T, 1, 4>(a, stream, syn);
    else if (dmax <= 8)
        launch_tma_d<T, 1, 8>(a, stream, syn);
    else if (dmax <= 12)
        launch_tma_d<T, 1, 12>(a, stream, syn);
    else if (dmax <= 16)
        launch_tma_d<T, 1, 16>(a, stream, syn);
    else
        launch_tma_d<T, 1, 32>(a, stream, syn);
}

static int dmax_bucket(int d) { return d <= 4 ? 4 : d <= 8 ? 8 : d <= 12 ? 12 : d <= 16 ? 16 : 32; }

static bool use_tma(const qcl_state *st) {
    // bulk copies move whole lane rows: W * sizeof(T) must be a 16-byte multiple; the flow
    // engine (4) uses these kernels for single layers and for codes/precisions it does not cover
    return (st->engine == 0 || st->engine == 4) && ((size_t)st->W * st->esz) % 16 == 0;
}

static void enqueue_unit_tma(qcl_state *st, const qcl_plan::Unit &u, cudaStream_t stream, double clip, double eps,
                             int g0, int ng) {
    const qcl_plan *p = st->plan;
    const int V = vec_width(st, u.dmax);
    const int D = dmax_bucket(u.dmax);
    PipeArgs a;
    a.r = slot_range(st, u.list_off, u.count, V, p->slot_list);
    a.r.g0 = g0;
    a.L = st->L;
    a.R = st->R;
    a.syn = st->has_syn ? st->syn : nullptr;
    a.KT = pipe_warps() * 32 * V / st->W;  // one (check, V lanes) item per consumer thread
    a.kblocks = (int)cdiv(p->z, a.KT);
    a.tiles = (int64_t)ng * u.count * a.kblocks;
    // ring depth: QCL_PIPE_STAGES, default 3 (capped so the ring fits ~112 KB)
    {
        static int want = env_int("QCL_PIPE_STAGES", 3);
        const size_t stage_bytes = (size_t)2 * D * pipe_warps() * 32 * V * st->esz;
        int s_ = std::max(2, std::min(want, (int)kMaxStages));
        while (s_ > 2 && s_ * stage_bytes > 112 * 1024) s_--;
        a.stages = s_;
    }
    a.uniform = p->layer_uniform[u.layer];
    a.n_active = st->g_et ? st->n_active : nullptr;
    // |r| <= Phi(eps) (the largest Phi value), so the r clip only binds for small clips
    a.clip_r = clip <= 1.001 * log1p(2.0 / expm1(eps));
    a.clip = clip;
    a.eps = eps;
    a.mag_max = mag_bound(clip, eps);
    if (st->prec == QCL_PREC_FP32)
        launch_tma<float>(a, V, u.dmax, stream, st->has_syn);
    else
        launch_tma<double>(a, V, u.dmax, stream, st->has_syn);
    st->launches_layer++;
    st->launches_all++;
}

static void enqueue_unit(qcl_state *st, const qcl_plan::Unit &u, cudaStream_t stream, double clip, double eps,
                         int g0, int ng) {
    // the TMA ring needs two stages of 2*D*KT*W elements in shared memory; wide FP64 rows
    // (row degree > 16: 2 x 128 KB) do not fit and run on the direct kernel
    const bool tma_fits = (size_t)2 * 2 * dmax_bucket(u.dmax) * pipe_warps() * 32 * vec_width(st, u.dmax) * st->esz +
                              128 <= 227 * 1024;
    if (use_tma(st) && tma_fits) {
        enqueue_unit_tma(st, u, stream, clip, eps, g0, ng);
        return;
    }
    const qcl_plan *p = st->plan;
    const int V = vec_width(st, u.dmax);
    LayerArgs a;
    a.r = slot_range(st, u.list_off, u.count, V, p->slot_list);
    a.r.g0 = g0;
    a.L = st->L;
    a.R = st->R;
    a.syn = st->has_syn ? st->syn : nullptr;
    a.uniform = p->layer_uniform[u.layer];
    a.clip_r = clip <= 1.001 * log1p(2.0 / expm1(eps));  // |r| <= Phi(eps)
    a.n_active = st->g_et ? st->n_active : nullptr;
    a.clip = clip;
    a.eps = eps;
    a.mag_max = mag_bound(clip, eps);
    dim3 grid((unsigned)((int64_t)ng * a.r.nslots * a.r.bps));
    if (st->prec == QCL_PREC_FP32) {
        if (V == 4)
            launch_layer_v<float, 4>(a, u.dmax, grid, stream, st->has_syn);
        else if (V == 2)
            launch_layer_v<float, 2>(a, u.dmax, grid, stream, st->has_syn);
        else
            launch_layer_v<float, 1>(a, u.dmax, grid, stream, st->has_syn);
    } else {
        if (V == 2)
            launch_layer_v<double, 2>(a, u.dmax, grid, stream, st->has_syn);
        else
            launch_layer_v<double, 1>(a, u.dmax, grid, stream, st->has_syn);
    }
    st->launches_layer++;
    st->launches_all++;
}

// One merged layer for lane groups [g0, g0 + ng): its launch units are independent
// (disjoint columns), so with fork != 0 units after the first run on side streams
// forked from / joined back into `stream` (parallel branches in the sweep graph).
static void enqueue_layer(qcl_state *st, int layer, double clip, double eps, cudaStream_t stream, int g0, int ng,
                          bool fork) {
    const qcl_plan *p = st->plan;
    const int u0 = p->layer_unit0[layer], u1 = p->layer_unit0[layer + 1];
    if (!fork || u1 - u0 == 1) {
        for (int u = u0; u < u1; u++) enqueue_unit(st, p->units[u], stream, clip, eps, g0, ng);
        return;
    }
    cudaEventRecord(st->fork, stream);
    for (int u = u0 + 1; u < u1; u++) {
        cudaStream_t side = st->side[(u - u0 - 1) % kSideStreams];
        cudaStreamWaitEvent(side, st->fork, 0);
        enqueue_unit(st, p->units[u], side, clip, eps, g0, ng);
    }
    enqueue_unit(st, p->units[u0], stream, clip, eps, g0, ng);
    for (int u = u0 + 1; u < u1; u++) {
        const int i = (u - u0 - 1) % kSideStreams;
        if (u + kSideStreams < u1) continue;  // only the last unit on each side stream joins
        cudaEventRecord(st->join[i], st->side[i]);
        cudaStreamWaitEvent(stream, st->join[i], 0);
    }
}

// Independent chains: lane groups never interact, so the sweep of each chain of groups
// is its own sequence of layer launches on its own stream.  Chains run concurrently,
// and one chain's kernels fill the ramp-up/tail of another's (the per-launch fixed cost
// is ~17% of a 64-codeword sweep with a single chain).
static int n_chains(const qcl_state *st) {
    // 2 chains measured best for 64-128 codewords (tools/chain_sweep.sh, profiles/README.md)
    static int env = env_int("QCL_CHAINS", 2);
    int c = env > 0 ? env : st->G;
    return std::max(1, std::min({c, st->G, kSideStreams}));
}

static void enqueue_sweep(qcl_state *st, double clip, double eps) {
    const qcl_plan *p = st->plan;
    const int chains = n_chains(st);
    if (chains == 1) {
        for (int l = 0; l < p->n_layers; l++) enqueue_layer(st, l, clip, eps, st->stream, 0, st->G, true);
        return;
    }
    cudaEventRecord(st->fork, st->stream);
    for (int c = 0; c < chains; c++) {
        const int g0 = (int)((int64_t)st->G * c / chains), g1 = (int)((int64_t)st->G * (c + 1) / chains);
        cudaStream_t cs = c == 0 ? st->stream : st->side[c - 1];
        if (c) cudaStreamWaitEvent(cs, st->fork, 0);
        for (int l = 0; l < p->n_layers; l++) enqueue_layer(st, l, clip, eps, cs, g0, g1 - g0, false);
    }
    for (int c = 1; c < chains; c++) {
        cudaEventRecord(st->join[c - 1], st->side[c - 1]);
        cudaStreamWaitEvent(st->stream, st->join[c - 1], 0);
    }
}

// ------------------------------------------------- persistent per-layer engine (W <= 2)
// One or two codewords (BASELINE configs[1]) run on the direct per-layer kernels, ~33
// dependent launches per sweep.  layer_persist_kernel (kernels.cuh) runs every sweep of
// the decode in ONE cooperative launch with a grid barrier between launch units; the
// per-thread arithmetic is layer_tile, shared with layer_kernel, so the result is
// bit-identical.  QCL_PERSIST=0 selects the per-layer launches.
static size_t persist_smem(const qcl_state *st);
static bool use_persist(const qcl_state *st) {
    // engines 0 / 4 where the lane rows are too narrow for bulk copies (engine 1 keeps the
    // per-layer launches).  QCL_PERSIST: 1 (default) where it measured faster -- FP64 and
    // two lanes (one codeword FP64 16.57 -> 14.59 ms, two FP32 5.28 -> 4.89 ms); one FP32
    // codeword measured 4.44-4.60 ms persistent against 4.42-4.46 per-layer on different
    // boxes, so it keeps the per-layer graph; 2: every 1-2 lane decode; 0: never.
    static const int mode = env_int("QCL_PERSIST", 1);
    const bool fits = (st->engine == 0 || st->engine == 4) && st->W <= 2 && !use_tma(st) && !st->msg16 &&
                      persist_smem(st) <= 160 * 1024;
    return fits && (mode == 2 || (mode == 1 && (st->prec == QCL_PREC_FP64 || st->W == 2)));
}

template <typename T, bool SYN>
static void (*persist_kernel(int maxd))(PersistArgs) {
    switch (maxd) {
        case 4: return layer_persist_kernel<T, SYN, 4>;
        case 8: return layer_persist_kernel<T, SYN, 8>;
        case 12: return layer_persist_kernel<T, SYN, 12>;
        case 16: return layer_persist_kernel<T, SYN, 16>;
        default: return layer_persist_kernel<T, SYN, 32>;
    }
}
static void (*persist_kernel(const qcl_state *st))(PersistArgs) {
    if (st->prec == QCL_PREC_FP32)
        return st->has_syn ? persist_kernel<float, true>(st->p_maxd) : persist_kernel<float, false>(st->p_maxd);
    return st->has_syn ? persist_kernel<double, true>(st->p_maxd) : persist_kernel<double, false>(st->p_maxd);
}

constexpr size_t kPersistBarBytes = 128 * (5 + 1024);  // barrier word, arrivals, one line per CTA (<= 1024)
static int persist_threads() {
    static const int t = env_int("QCL_PERSIST_THREADS", 256) == 512 ? 512 : 256;
    return t;
}
static size_t persist_smem(const qcl_state *st) {
    const qcl_plan *p = st->plan;
    return persist_smem_bytes((int)p->units.size(), p->S, p->E, (int)p->h_slot_list.size());
}

static int persist_grid(const qcl_state *st, int max_blocks) {
    int sms = 0, per_sm = 0;
    const size_t smem = persist_smem(st);
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st->plan->device));
    CK(cudaFuncSetAttribute(persist_kernel(st), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persist_kernel(st), persist_threads(), smem));
    if (per_sm < 1) return 0;
    // one CTA per SM and lane (tools/persist_sweep.sh: B = 1 4.52 ms at one CTA per SM
    // against 4.66 at two; B = 2 4.95 against 5.50)
    static const int cap = env_int("QCL_PERSIST_CTAS_PER_SM", 0);
    per_sm = std::min(per_sm, cap > 0 ? cap : st->W);
    const int halves = persist_threads() / kBlock;
    return std::max(1, std::min({(max_blocks + halves - 1) / halves, sms * per_sm, 1024}));
}

// Unit table of one sweep for (clip, eps, syndrome presence); uploaded outside any graph
// capture on the state's stream and waited for there.
static int ensure_persist(qcl_state *st, double clip, double eps) {
    if (st->punits && st->p_clip == clip && st->p_eps == eps && st->p_syn == st->has_syn) return QCL_OK;
    const qcl_plan *p = st->plan;
    std::vector<PersistUnit> units;
    int max_blocks = 1, maxd = 4;
    for (const auto &u : p->units) {
        PersistUnit pu{};
        LayerArgs &a = pu.a;
        a.r = slot_range(st, u.list_off, u.count, 1, p->slot_list);
        a.r.g0 = 0;
        a.L = st->L;
        a.R = st->R;
        a.syn = st->has_syn ? st->syn : nullptr;
        a.uniform = p->layer_uniform[u.layer];
        a.clip_r = clip <= 1.001 * log1p(2.0 / expm1(eps));
        a.n_active = nullptr;
        a.clip = clip;
        a.eps = eps;
        a.mag_max = mag_bound(clip, eps);
        pu.blocks = (int32_t)((int64_t)st->G * a.r.nslots * a.r.bps);
        pu.dcls = dmax_bucket(u.dmax);
        pu.layer = u.layer;
        maxd = std::max(maxd, pu.dcls);
        max_blocks = std::max(max_blocks, pu.blocks);
        units.push_back(pu);
    }
    CK(cudaStreamSynchronize(st->stream));  // a previous decode may still read the old table
    if (!st->punits || st->p_nu < (int)units.size()) {
        if (st->punits) cudaFree(st->punits);
        st->punits = nullptr;
        CK(cudaMalloc(&st->punits, sizeof(PersistUnit) * units.size()));
    }
    if (!st->pbar) CK(cudaMalloc(&st->pbar, kPersistBarBytes));
    CK(cudaMemcpyAsync(st->punits, units.data(), sizeof(PersistUnit) * units.size(), cudaMemcpyHostToDevice,
                       st->stream));
    CK(cudaStreamSynchronize(st->stream));
    st->p_nu = (int)units.size();
    st->p_maxd = maxd;
    st->p_grid = persist_grid(st, max_blocks);
    if (st->p_grid <= 0) return fail(QCL_ECUDA, "persistent engine: no occupancy");
    st->p_clip = clip;
    st->p_eps = eps;
    st->p_syn = st->has_syn;
    return QCL_OK;
}

// `sweeps` sweeps in one cooperative launch (all CTAs co-resident: the grid barrier
// cannot deadlock, also next to other work on the device).
static int enqueue_persist(qcl_state *st, int sweeps, bool et) {
    const qcl_plan *p = st->plan;
    CK(cudaMemsetAsync(st->pbar, 0, kPersistBarBytes, st->stream));
    PersistArgs pa;
    pa.units = st->punits;
    pa.nu = st->p_nu;
    pa.S = p->S;
    pa.E = p->E;
    pa.nlist = (int)p->h_slot_list.size();
    pa.slots = p->slots;
    pa.edges = p->edges;
    pa.slot_list = p->slot_list;
    pa.sweeps = sweeps;
    pa.bar = st->pbar;
    pa.n_active = et ? st->n_active : nullptr;
    static const int bar_mode = env_int("QCL_PERSIST_BAR", 1);  // 1 measured best (DESIGN 3.4)
    pa.bar_mode = bar_mode;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)st->p_grid);
    cfg.blockDim = dim3(persist_threads());
    cfg.dynamicSmemBytes = persist_smem(st);
    cfg.stream = st->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, persist_kernel(st), pa));
    st->launches_layer++;
    st->launches_all++;
    return QCL_OK;
}

// ------------------------------------------------------------ flow engine (engine 4)
// One persistent launch runs many sweeps; tiles are ordered by completion flags
// (csrc/flow.cuh).  FP32 only, row degree <= 12, and W >= 4 lanes (16-byte bulk runs).
static bool use_flow(const qcl_state *st) {
    return st->engine == 4 && st->prec == QCL_PREC_FP32 && st->plan->flow_ok && st->plan->max_degree <= 12 &&
           st->W >= 4 && st->f_grid >= 0;
}

// FP16 edge messages exist only in the flow kernel's message path.
static int msg16_unsupported(const qcl_state *st, const char *what) {
    return fail(QCL_EUNSUP, "16-bit edge messages (QCL_PREC_FP32_MSG16) run on the flow engine only: %s "
                "(engine %d, max row degree %d, %d lanes)", what, st->engine, st->plan->max_degree, st->W);
}

// Tiling (per slot), the item list of one sweep and the flag/counter buffers.
static int ensure_flow(qcl_state *st, int counters) {
    const qcl_plan *p = st->plan;
    if (!st->fslot_tab) {
        std::vector<uint2> stab(p->S);
        std::vector<int> nkb(p->S);
        int32_t off = 0;
        for (int s = 0; s < p->S; s++) {
            const int d = p->h_slots[s].degree;
            const uint32_t cls = d <= 4 ? 0 : d <= 8 ? 1 : 2;
            const int KT = flow_KT((int)cls, st->W);
            nkb[s] = (int)cdiv(p->z, KT);
            stab[s].x = (uint32_t)p->h_slots[s].edge_off | ((uint32_t)d << 16) | (cls << 24);
            stab[s].y = (uint32_t)off;
            off += nkb[s];
        }
        st->f_nkb_total = off;
        // item order (flow.cuh): group block, iteration, layer, lane group, slot, k-block.
        // Large batches run as blocks of 8 lane groups (64 codewords at W = 8), one block
        // after the other inside the same launch, so the L2-resident working set (the hot
        // columns' posteriors) stays that of 64 codewords: 128 codewords 51.9 -> 46.2 ms,
        // 256: 114 -> 96 ms (DESIGN 3.1).  QCL_FLOW_BLOCK_GROUPS: groups per block (0: one).
        static const int blk_groups = env_int("QCL_FLOW_BLOCK_GROUPS", 8);
        const int GB = (blk_groups > 0 && st->G > blk_groups && st->G % blk_groups == 0) ? blk_groups : st->G;
        st->f_nblk = st->G / GB;
        std::vector<int2> items;
        for (int b = 0; b < st->f_nblk; b++)
            for (int l = 0; l < p->n_layers; l++)
                for (int g = b * GB; g < (b + 1) * GB; g++)
                    for (int s = p->layer_start[l]; s < p->layer_start[l + 1]; s++)
                        for (int kb = 0; kb < nkb[s]; kb++) items.push_back(make_int2(s | (g << 16), kb));
        st->f_sweep_items = (int64_t)items.size() / st->f_nblk;
        CK(cudaMalloc(&st->fslot_tab, sizeof(uint2) * p->S));
        CK(cudaMemcpyAsync(st->fslot_tab, stab.data(), sizeof(uint2) * p->S, cudaMemcpyHostToDevice, st->stream));
        CK(cudaMalloc(&st->fitems, sizeof(int2) * items.size()));
        CK(cudaMemcpyAsync(st->fitems, items.data(), sizeof(int2) * items.size(), cudaMemcpyHostToDevice,
                           st->stream));
        CK(cudaMalloc(&st->fflags, sizeof(int) * QCL_FLAG_STRIDE * (size_t)st->G * st->f_nkb_total));
        if (env_int("QCL_FLOW_STATS", 0)) {
            CK(cudaMalloc(&st->fstats, 16 * sizeof(unsigned long long)));
            CK(cudaMemsetAsync(st->fstats, 0, 16 * sizeof(unsigned long long), st->stream));
        }
        // the uploads are on the state's stream (a device-wide synchronisation would be
        // illegal while another host thread captures a decode graph): wait for them here
        CK(cudaStreamSynchronize(st->stream));
        // ring depth: QCL_FLOW_STAGES (default 3 with two CTAs per SM, 5 with one), reduced
        // until the CTAs fit
        static int want = env_int("QCL_FLOW_STAGES", kFlowCtasPerSm == 1 ? 5 : 3);
        int stages = std::max(2, std::min(want, kFlowMaxStages));
        int sms = 0, per_sm = 0, max_smem = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
        CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device));
        while (stages > 2 && flow_smem_bytes(p->S, p->E, stages) * kFlowCtasPerSm + 1024 * kFlowCtasPerSm > 233472)
            stages--;
        const size_t smem = flow_smem_bytes(p->S, p->E, stages);
        if ((int64_t)smem > max_smem) {
            st->f_grid = -1;  // tables too large: the per-layer engine runs instead
            return QCL_OK;
        }
        st->f_stages = stages;
        for (auto kern : {flow_kernel<false, false>, flow_kernel<true, false>, flow_kernel<false, true>,
                          flow_kernel<true, true>, flow_kernel<false, false, __half>, flow_kernel<true, false, __half>,
                          flow_kernel<false, true, __half>, flow_kernel<true, true, __half>,
                          flow_kernel<false, false, float, true>, flow_kernel<true, false, float, true>,
                          flow_kernel<false, false, __half, true>, flow_kernel<true, false, __half, true>})
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel<false, false>, kFlowThreads, smem));
        st->f_grid = sms * std::max(1, per_sm);
    }
    if (st->f_counter_cap < counters) {
        if (st->fcounters) cudaFree(st->fcounters);
        st->fcounters = nullptr;
        st->f_counter_cap = 0;
        CK(cudaMalloc(&st->fcounters, sizeof(int) * counters));
        st->f_counter_cap = counters;
    }
    return QCL_OK;
}

// Fused early termination (flow.cuh): ET decodes on the flow engine run every sweep in one
// launch, with the per-sweep check as items of the same stream.  Needs W <= 8 (one byte of
// lane bits per variable); the frame pool keeps its per-sweep launches (lanes refill).
// QCL_FLOW_ET_FUSED=0: the per-sweep launch plus check kernels of round 1.
static bool use_flow_et(const qcl_state *st) {
    static const bool on = env_int("QCL_FLOW_ET_FUSED", 1) != 0;
    return on && use_flow(st) && st->W <= 8 && !st->pool_active;
}

static int ensure_flow_et(qcl_state *st) {
    const qcl_plan *p = st->plan;
    if (st->fitems_et) return QCL_OK;
    static const int blk_groups = env_int("QCL_FLOW_BLOCK_GROUPS", 8);
    const int GB = st->G / st->f_nblk;
    (void)blk_groups;
    // per group block: the sweep table -- layers 0..Lc, the check items of the PREVIOUS sweep
    // (one per lane group and layer: slots [s0, s1) as {s0 | g << 16, -1 - s1}), the other
    // layers -- then a tail with the last sweep's check items (flow.cuh flow_item_map)
    const int Lc = std::min(1, p->n_layers - 1);
    std::vector<int2> items, checks;
    for (int b = 0; b < st->f_nblk; b++) {
        checks.clear();
        for (int g = b * GB; g < (b + 1) * GB; g++)
            for (int l = 0; l < p->n_layers; l++)
                checks.push_back(make_int2(p->layer_start[l] | (g << 16), -1 - p->layer_start[l + 1]));
        for (int l = 0; l < p->n_layers; l++) {
            for (int g = b * GB; g < (b + 1) * GB; g++)
                for (int s = p->layer_start[l]; s < p->layer_start[l + 1]; s++) {
                    const int d = p->h_slots[s].degree;
                    const int KT = flow_KT(d <= 4 ? 0 : d <= 8 ? 1 : 2, st->W);
                    for (int kb = 0; kb < (int)cdiv(p->z, KT); kb++) items.push_back(make_int2(s | (g << 16), kb));
                }
            if (l == Lc) items.insert(items.end(), checks.begin(), checks.end());
        }
        items.insert(items.end(), checks.begin(), checks.end());  // tail
    }
    st->f_check_items = p->n_layers;
    st->f_sweep_items_et = (int64_t)items.size() / st->f_nblk - (int64_t)GB * p->n_layers;
    CK(cudaMalloc(&st->fitems_et, sizeof(int2) * items.size()));
    CK(cudaMemcpyAsync(st->fitems_et, items.data(), sizeof(int2) * items.size(), cudaMemcpyHostToDevice,
                       st->stream));
    CK(cudaMalloc(&st->fsnap, (size_t)2 * st->G * p->n));
    CK(cudaMalloc(&st->fsign, (size_t)st->G * p->n));
    CK(cudaMalloc(&st->fet, sizeof(int) * 5 * QCL_FLAG_STRIDE * (size_t)st->G));
    CK(cudaMalloc(&st->famask, sizeof(uint32_t) * st->G));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

// Last sweep of a fused no-ET decode, or -1 with QCL_FLOW_DEFER=0 (degree-1 deferral off).
static int flow_defer_last(int max_iterations) {
    static int on = env_int("QCL_FLOW_DEFER", 1);
    return on ? max_iterations - 1 : -1;
}

// Flags and claim counters back to zero: the start of a flow decode (sweep 0).
static int enqueue_flow_reset(qcl_state *st, int counters) {
    int rc = ensure_flow(st, counters);
    if (rc) return rc;
    CK(cudaMemsetAsync(st->fflags, 0, sizeof(int) * QCL_FLAG_STRIDE * (size_t)st->G * st->f_nkb_total, st->stream));
    CK(cudaMemsetAsync(st->fcounters, 0, sizeof(int) * counters, st->stream));
    return QCL_OK;
}

// Sweeps [t0, t0 + T) in one persistent launch using claim counter `counter`.
static int enqueue_flow(qcl_state *st, double clip, double eps, int t0, int T, int counter, bool et,
                        int defer_last = -1, const int *t_dev = nullptr, int fresh_t = -1, bool etf = false) {
    const qcl_plan *p = st->plan;
    FlowArgs a = {};
    const int64_t sweep_items = etf ? st->f_sweep_items_et : st->f_sweep_items;
    a.slot_tab = st->fslot_tab;
    a.edge_tab = p->fedge_tab;
    a.items = etf ? st->fitems_et : st->fitems;
    a.sweep_items = (int32_t)sweep_items;
    flow_sweep_divisor((uint32_t)sweep_items, a.sweep_mul, a.sweep_shift);
    const int64_t tail = etf ? (int64_t)(st->G / st->f_nblk) * st->f_check_items : 0;
    a.blk_items = (int32_t)(T * sweep_items + tail);
    flow_sweep_divisor((uint32_t)a.blk_items, a.blk_mul, a.blk_shift);
    a.item_end = (int32_t)(st->f_nblk * a.blk_items);
    a.tab_stride = (int32_t)(sweep_items + tail);
    a.sweeps = T;
    a.check_items = st->f_check_items;
    if (etf) {
        const size_t gs = (size_t)st->G * QCL_FLAG_STRIDE;
        a.snap = st->fsnap;
        a.fsign = st->fsign;
        a.cdone = st->fet;
        a.decided = st->fet + gs;
        a.unsat = reinterpret_cast<uint32_t *>(st->fet + 2 * gs);
        a.amask = st->famask;
        a.conv = st->conv;
        a.iters = st->iters;
        a.synpack = st->has_syn ? st->synpack : nullptr;
    }
    a.G = st->G;
    a.slot_mask = p->fslast;
    a.t_base = t0;
    a.t_dev = t_dev;
    a.fresh_t = fresh_t;
    a.counter = st->fcounters + counter;
    a.flags = st->fflags;
    a.nkb_total = st->f_nkb_total;
    a.L = st->L;
    a.R = st->R;
    a.syn = st->has_syn ? st->syn : nullptr;
    a.n = p->n;
    a.E = p->E;
    a.S = p->S;
    a.z = p->z;
    a.lw = st->lw;
    a.stages = st->f_stages;
    a.clip_r = clip <= 1.001 * log1p(2.0 / expm1(eps));  // |r| <= Phi(eps)
    a.n_active = et ? st->n_active : nullptr;
    a.gactive = et ? st->gactive : nullptr;
    a.defer_last = defer_last;
    a.fresh = st->pool_active ? st->pfresh : nullptr;
    a.stats = st->fstats;
    a.clip = clip;
    a.eps = eps;
    a.mag_max = mag_bound(clip, eps);
    a.clip_f = (float)clip;
    a.mag_f = (float)a.mag_max;
    const size_t smem = flow_smem_bytes(p->S, p->E, st->f_stages);
    const int64_t grid = std::min<int64_t>(st->f_grid, a.item_end);
    const bool prof = st->fstats != nullptr;
    void (*kern)(FlowArgs);
    if (etf)  // fused early termination (no instrumented variant)
        kern = st->msg16 ? (st->has_syn ? flow_kernel<true, false, __half, true> : flow_kernel<false, false, __half, true>)
                         : (st->has_syn ? flow_kernel<true, false, float, true> : flow_kernel<false, false, float, true>);
    else if (st->msg16)
        kern = st->has_syn ? (prof ? flow_kernel<true, true, __half> : flow_kernel<true, false, __half>)
                           : (prof ? flow_kernel<false, true, __half> : flow_kernel<false, false, __half>);
    else
        kern = st->has_syn ? (prof ? flow_kernel<true, true> : flow_kernel<true, false>)
                           : (prof ? flow_kernel<false, true> : flow_kernel<false, false>);
    if (flow_static(etf)) {  // static item order: all CTAs must be co-resident
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(kFlowThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
        kern<<<(unsigned)grid, kFlowThreads, smem, st->stream>>>(a);
    }
    CK(cudaGetLastError());
    st->launches_layer++;
    st->launches_all++;
    return QCL_OK;
}

// Hard decisions of every lane packed into sign words (decoder.py:264-266).
static int enqueue_signs(qcl_state *st, const uint8_t *gact = nullptr) {
    const qcl_plan *p = st->plan;
    const int64_t Gn = (int64_t)st->G * p->n;
    const unsigned grid = (unsigned)cdiv(Gn, kBlock);
#ifndef QCL_SIGN_PER_VAR
#define QCL_SIGN_PER_VAR 1
#endif
    if (st->prec == QCL_PREC_FP32 && QCL_SIGN_PER_VAR)
        sign_pack_var_kernel<float><<<(unsigned)cdiv(p->n, kBlock), kBlock, 0, st->stream>>>(
            (const float *)st->L, st->G, st->lw, st->signs, p->n, gact);
    else if (st->prec == QCL_PREC_FP32)
        sign_pack_kernel<float><<<grid, kBlock, 0, st->stream>>>((const float *)st->L, Gn, st->lw, st->signs, p->n,
                                                                  gact);
    else
        sign_pack_kernel<double><<<grid, kBlock, 0, st->stream>>>((const double *)st->L, Gn, st->lw, st->signs,
                                                                   p->n, gact);
    st->launches_all++;
    CK(cudaGetLastError());
    return QCL_OK;
}

// syndrome_satisfied for every codeword (decoder.py:268-273) -> st->unsat lane masks;
// with gact, lane groups whose frames have all converged are skipped.
static int enqueue_check(qcl_state *st, const uint8_t *gact = nullptr) {
    const qcl_plan *p = st->plan;
    int rc = enqueue_signs(st, gact);
    if (rc) return rc;
    CK(cudaMemsetAsync(st->unsat, 0, sizeof(uint32_t) * st->G, st->stream));
    const int64_t total = (int64_t)p->S * p->z;
    check_packed_kernel<<<(unsigned)cdiv(total, kBlock), kBlock, 0, st->stream>>>(
        p->slots, p->edges, p->n, p->S, p->z, st->G, st->signs, st->has_syn ? st->synpack : nullptr, st->unsat, gact);
    st->launches_all++;
    CK(cudaGetLastError());
    return QCL_OK;
}

static void enqueue_group_active(qcl_state *st) {
    group_active_kernel<<<(unsigned)cdiv(st->G, kBlock), kBlock, 0, st->stream>>>(st->Bp, st->lw, st->active,
                                                                                    st->gactive);
    st->launches_all++;
}

// Words (B, n) for codewords with take[b] from the packed signs of the last check.
static int enqueue_words(qcl_state *st, const uint8_t *take) {
    const qcl_plan *p = st->plan;
    words_from_signs_kernel<<<(unsigned)cdiv(p->n, kBlock), kBlock, 0, st->stream>>>(st->signs, p->n, st->lw, st->B,
                                                                                     take, st->words);
    st->launches_all++;
    CK(cudaGetLastError());
    return QCL_OK;
}

static int enqueue_syn_pack(qcl_state *st) {
    const qcl_plan *p = st->plan;
    const int64_t words = (int64_t)st->G * p->S * p->z;
    syn_pack_kernel<<<(unsigned)cdiv(words, kBlock), kBlock, 0, st->stream>>>(st->syn, words, st->lw,
                                                                               (int64_t)p->S * p->z, st->synpack);
    CK(cudaGetLastError());
    return QCL_OK;
}

// One sweep over every layer, captured once into a graph and replayed per iteration.
static int run_sweep(qcl_state *st, double clip, double eps, bool et) {
    if (!st->sweep_exec || st->g_clip != clip || st->g_eps != eps || st->g_syn != st->has_syn || st->g_et != et) {
        st->g_et = et;
        if (st->sweep_exec) {
            cudaGraphExecDestroy(st->sweep_exec);
            st->sweep_exec = nullptr;
        }
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(st->stream, cudaStreamCaptureModeThreadLocal));
        const int64_t saved = st->launches_layer, saved_all = st->launches_all;
        enqueue_sweep(st, clip, eps);
        st->sweep_launches = st->launches_layer - saved;
        st->launches_layer = saved;
        st->launches_all = saved_all;
        CK(cudaStreamEndCapture(st->stream, &graph));
        cudaError_t e = cudaGraphInstantiate(&st->sweep_exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(e);
        st->g_clip = clip;
        st->g_eps = eps;
        st->g_syn = st->has_syn;
        st->g_et = et;
    }
    if (st->profiling) {
        // CUDA events on the launching stream around each sweep (30 layer kernels for the
        // rate-0.1 code); read after the decode's final sync, so no host stall is added
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st->stream));
        CK(cudaGraphLaunch(st->sweep_exec, st->stream));
        CK(cudaEventRecord(b, st->stream));
        st->sweep_events.push_back({a, b});
    } else {
        CK(cudaGraphLaunch(st->sweep_exec, st->stream));
    }
    st->launches_layer += st->sweep_launches;
    st->launches_all += st->sweep_launches;
    return QCL_OK;
}

// ----------------------------------------------------------------------------- C ABI

extern "C" {

int32_t qcl_abi_version(void) { return 1; }

const char *qcl_last_error(void) { return g_err.c_str(); }

int qcl_device_count(int32_t *count) {
    int c = 0;
    CK(cudaGetDeviceCount(&c));
    *count = c;
    return QCL_OK;
}

int qcl_plan_create(int32_t z, int32_t n_cols, int32_t n_slots, int32_t n_layers, int32_t n_edges,
                    const int32_t *edge_shift, const int32_t *edge_col, const int32_t *slot_offsets,
                    const int32_t *slot_rows, const int32_t *layer_slot_starts,
                    const int32_t *schedule_rows, int32_t device, qcl_plan **out) {
    if (!out) return fail(QCL_EVALUE, "out is NULL");
    *out = nullptr;
    if (z < 1 || n_cols < 1 || n_slots < 1 || n_layers < 1 || n_edges < 1)
        return fail(QCL_EVALUE, "empty code");
    // decoder.py:118-120
    for (int s = 0; s < n_slots; s++)
        if (schedule_rows[s] != slot_rows[s])
            return fail(QCL_EVALUE, "schedule does not match the compact index row order");
    if (layer_slot_starts[0] != 0 || layer_slot_starts[n_layers] != n_slots)
        return fail(QCL_EVALUE, "schedule does not match the compact index row order");
    if (slot_offsets[0] != 0 || slot_offsets[n_slots] != n_edges)
        return fail(QCL_EVALUE, "slot offsets do not cover the edge list");
    auto p = new qcl_plan();
    p->device = device;
    p->z = z;
    p->n_cols = n_cols;
    p->S = n_slots;
    p->n_layers = n_layers;
    p->E = n_edges;
    p->n = (int64_t)n_cols * z;
    p->m = (int64_t)n_slots * z;
    p->layer_start.assign(layer_slot_starts, layer_slot_starts + n_layers + 1);
    std::vector<EdgeInfo> h_edges(n_edges);
    for (int e = 0; e < n_edges; e++) {
        if (edge_col[e] < 0 || edge_col[e] >= n_cols || edge_shift[e] < 0 || edge_shift[e] >= z) {
            delete p;
            return fail(QCL_EVALUE, "edge %d out of range", e);
        }
        h_edges[e] = EdgeInfo{edge_col[e] * z, edge_shift[e], 0, 0};
    }
    {
        std::vector<int> coldeg(n_cols, 0);
        for (int e = 0; e < n_edges; e++) coldeg[edge_col[e]]++;
        for (int e = 0; e < n_edges; e++) h_edges[e].reused = coldeg[edge_col[e]] > 1;
    }
    p->h_slots.resize(n_slots);
    for (int s = 0; s < n_slots; s++) {
        int d = slot_offsets[s + 1] - slot_offsets[s];
        if (d < 1) {
            delete p;
            return fail(QCL_EVALUE, "empty check row");
        }
        p->h_slots[s] = SlotInfo{slot_offsets[s], d, slot_rows[s], 0};
        p->max_degree = std::max(p->max_degree, d);
    }
    if (p->max_degree > 32) {
        delete p;
        return fail(QCL_EUNSUP, "row degree %d > 32 is not supported by this build", p->max_degree);
    }
    // decoder.py:144-154: rows merged into one layer must touch disjoint columns
    for (int l = 0; l < n_layers; l++) {
        std::set<int> seen;
        int dmax = 0, d0 = -1, uniform = 1;
        for (int s = layer_slot_starts[l]; s < layer_slot_starts[l + 1]; s++) {
            std::set<int> cols;
            for (int e = slot_offsets[s]; e < slot_offsets[s + 1]; e++) cols.insert(edge_col[e]);
            for (int c : cols)
                if (seen.count(c)) {
                    delete p;
                    return fail(QCL_EVALUE, "rows within a layer share a base column");
                }
            seen.insert(cols.begin(), cols.end());
            int d = slot_offsets[s + 1] - slot_offsets[s];
            dmax = std::max(dmax, d);
            if (d0 < 0) d0 = d;
            if (d != d0) uniform = 0;
        }
        if (layer_slot_starts[l + 1] <= layer_slot_starts[l]) {
            delete p;
            return fail(QCL_EVALUE, "schedule contains an empty layer");
        }
        p->layer_dmax.push_back(dmax);
        p->layer_uniform.push_back(uniform);
    }
    {
        std::vector<int32_t> list;
        auto bucket = [](int d) { return d <= 4 ? 4 : d <= 8 ? 8 : d <= 12 ? 12 : d <= 16 ? 16 : 32; };
        for (int l = 0; l < n_layers; l++) {
            p->layer_unit0.push_back((int)p->units.size());
            for (int b : {4, 8, 12, 16, 32}) {
                qcl_plan::Unit u{l, (int)list.size(), 0, 0};
                for (int s = layer_slot_starts[l]; s < layer_slot_starts[l + 1]; s++) {
                    int d = slot_offsets[s + 1] - slot_offsets[s];
                    if (bucket(d) != b) continue;
                    list.push_back(s);
                    u.count++;
                    u.dmax = std::max(u.dmax, d);
                }
                if (u.count) p->units.push_back(u);
            }
        }
        p->layer_unit0.push_back((int)p->units.size());
        p->h_slot_list = list;
    }
    // flow engine: per circulant the previous writer of its column in cyclic schedule
    // (= slot) order; the first toucher of a column waits on the last one of the previous
    // iteration (itself for a degree-1 column).  Packed as in csrc/flow.cuh.
    std::vector<uint2> h_etab(n_edges);
    std::vector<uint32_t> h_slast(n_slots, 0u);
    p->flow_ok = z <= 65535 && n_cols <= 32767 && n_slots <= 32767 && n_edges <= 65535;
    {
        std::vector<std::vector<int>> touch(n_cols);  // circulants per column, slot order
        for (int e = 0; e < n_edges; e++) touch[edge_col[e]].push_back(e);
        std::vector<int> slot_of(n_edges);
        for (int s = 0; s < n_slots; s++)
            for (int e = slot_offsets[s]; e < slot_offsets[s + 1]; e++) slot_of[e] = s;
        for (int c = 0; c < n_cols; c++) {
            const auto &tl = touch[c];
            for (size_t i = 0; i < tl.size(); i++) {
                const int e = tl[i], pe = i ? tl[i - 1] : tl.back();
                int delta = edge_shift[e] - edge_shift[pe];
                delta += delta < 0 ? z : 0;
                const uint32_t reused = tl.size() > 1;
                h_etab[e].x = (uint32_t)(c & 0x7fff) | (reused << 15) | ((uint32_t)edge_shift[e] << 16);
                h_etab[e].y = (uint32_t)(slot_of[pe] & 0x7fff) | ((i == 0 ? 1u : 0u) << 15) | ((uint32_t)delta << 16);
                const int j = e - slot_offsets[slot_of[e]];
                if (j < 16 && i + 1 == tl.size()) h_slast[slot_of[e]] |= 1u << (16 + j);
                if (j < 16 && tl.size() == 1) h_slast[slot_of[e]] |= 1u << j;
            }
        }
    }
    DeviceScope dscope_(device);
    cudaError_t e = dscope_.ok ? cudaSuccess : cudaErrorInvalidDevice;
    // uploads on a private stream, waited for once (the plan is immutable afterwards and
    // states run on their own non-blocking streams); no device-wide synchronisation, which
    // is illegal while another host thread captures a decode graph
    cudaStream_t up = nullptr;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    auto put = [&](void *dst, const void *src, size_t bytes) {
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, up);
    };
    if (e == cudaSuccess) e = cudaMalloc(&p->fedge_tab, sizeof(uint2) * n_edges);
    put(p->fedge_tab, h_etab.data(), sizeof(uint2) * n_edges);
    if (e == cudaSuccess) e = cudaMalloc(&p->fslast, sizeof(uint32_t) * n_slots);
    put(p->fslast, h_slast.data(), sizeof(uint32_t) * n_slots);
    std::vector<int32_t> untouched;
    {
        std::vector<char> used(n_cols, 0);
        for (int i = 0; i < n_edges; i++) used[edge_col[i]] = 1;
        for (int c = 0; c < n_cols; c++)
            if (!used[c]) untouched.push_back(c);
    }
    p->n_untouched = (int)untouched.size();
    if (e == cudaSuccess && !untouched.empty()) e = cudaMalloc(&p->funtouched, sizeof(int32_t) * untouched.size());
    if (!untouched.empty()) put(p->funtouched, untouched.data(), sizeof(int32_t) * untouched.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->slot_list, sizeof(int32_t) * p->h_slot_list.size());
    put(p->slot_list, p->h_slot_list.data(), sizeof(int32_t) * p->h_slot_list.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->slots, sizeof(SlotInfo) * n_slots);
    if (e == cudaSuccess) e = cudaMalloc(&p->edges, sizeof(EdgeInfo) * n_edges);
    put(p->slots, p->h_slots.data(), sizeof(SlotInfo) * n_slots);
    put(p->edges, h_edges.data(), sizeof(EdgeInfo) * n_edges);
    if (up) {
        const cudaError_t e2 = cudaStreamSynchronize(up);
        if (e == cudaSuccess) e = e2;
        cudaStreamDestroy(up);
    }
    if (e != cudaSuccess) {
        cudaFree(p->slots);
        cudaFree(p->edges);
        cudaFree(p->slot_list);
        cudaFree(p->fedge_tab);
        cudaFree(p->fslast);
        cudaFree(p->funtouched);
        delete p;
        return fail(QCL_ECUDA, "plan upload failed: %s", cudaGetErrorString(e));
    }
    *out = p;
    return QCL_OK;
}

int qcl_state_destroy(qcl_state *st);

int qcl_plan_destroy(qcl_plan *p) {
    if (!p) return QCL_OK;
    DeviceScope dscope_(p->device);
    for (auto *s : p->cache) qcl_state_destroy(s);
    cudaFree(p->slots);
    cudaFree(p->edges);
    cudaFree(p->slot_list);
    cudaFree(p->fedge_tab);
    cudaFree(p->fslast);
    cudaFree(p->funtouched);
    delete p;
    return QCL_OK;
}

int qcl_plan_info(const qcl_plan *p, int64_t *n_vars, int64_t *n_checks, int64_t *n_edges_expanded,
                  int32_t *n_layers, int32_t *max_degree) {
    if (!p) return fail(QCL_EVALUE, "plan is NULL");
    if (n_vars) *n_vars = p->n;
    if (n_checks) *n_checks = p->m;
    if (n_edges_expanded) *n_edges_expanded = (int64_t)p->E * p->z;
    if (n_layers) *n_layers = p->n_layers;
    if (max_degree) *max_degree = p->max_degree;
    return QCL_OK;
}

static int lanes_log2(int64_t B) {
    // W = min(8, next pow2 >= B): 8 lanes (32-byte FP32 runs, still whole 16-byte bulk-copy
    // units) give the flow engine 8 independent lane groups per 64 codewords, i.e. more
    // slack between a tile and the previous-layer tiles it waits for (tools/flow_grid.sh:
    // 25.7 ms at W = 8 vs 26.6 ms at W = 32 per 64-codeword decode); override: QCL_LANES
    const char *env = getenv("QCL_LANES");
    int want = env ? atoi(env) : 8;
    int lw = 0;
    while ((1 << lw) < B && (1 << lw) < want && lw < 5) lw++;
    return lw;
}

int qcl_state_create(qcl_plan *p, int64_t batch, int32_t precision, qcl_state **out) {
    if (!p || !out) return fail(QCL_EVALUE, "NULL argument");
    if (batch < 1) return fail(QCL_EVALUE, "batch must be at least 1");
    if (precision != QCL_PREC_FP32 && precision != QCL_PREC_FP64 && precision != QCL_PREC_FP32_MSG16)
        return fail(QCL_EVALUE, "unknown precision %d", precision);
    DEVICE_SCOPE(p->device);
    auto st = new qcl_state();
    st->plan = p;
    st->B = batch;
    st->api_prec = precision;
    st->msg16 = precision == QCL_PREC_FP32_MSG16;
    st->prec = st->msg16 ? QCL_PREC_FP32 : precision;
    st->esz = st->prec == QCL_PREC_FP32 ? 4 : 8;
    st->resz = st->msg16 ? 2 : st->esz;
    // FP16 runs of W lanes must stay whole 16-byte bulk-copy units: at least 8 lanes.
    // QCL_MIN_LANES=4 pads FP32 batches of 1-3 codewords to 4 lanes (idle lanes decode
    // zero LLRs) so that they run on the flow engine; off by default: one lane group has
    // no slack between dependent tiles, and the per-layer graph is faster there (B = 1:
    // 5.8 ms against 9.1 ms per 50-iteration decode, tools/latency_small_batch.py).
    static const int min_lanes_f32 = env_int("QCL_MIN_LANES", 1);
    const int lw_min = st->msg16 ? 3 : st->prec == QCL_PREC_FP32 ? (min_lanes_f32 >= 4 ? 2 : 0) : 0;
    st->lw = std::max(lw_min, lanes_log2(batch));
    st->W = 1 << st->lw;
    st->G = (int)cdiv(batch, st->W);
    st->Bp = (int64_t)st->G * st->W;
    if ((int64_t)st->G * p->S * p->z >= (1LL << 31) || st->Bp * p->n >= (1LL << 40)) {
        delete st;
        return fail(QCL_EUNSUP, "batch %lld too large for one state (split it across states)", (long long)batch);
    }
    const size_t nl = (size_t)st->Bp * p->n, ne = (size_t)st->Bp * p->E * p->z, nm = (size_t)st->Bp * p->m;
    cudaError_t e = cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking);
    for (int i = 0; i < kSideStreams && e == cudaSuccess; i++) {
        e = cudaStreamCreateWithFlags(&st->side[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->join[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->fork, cudaEventDisableTiming);
    auto al = [&](void **ptr, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(ptr, std::max<size_t>(bytes, 16));
    };
    al(&st->llr, nl * st->esz);
    al(&st->L, nl * st->esz);
    al(&st->R, ne * st->resz);
    al((void **)&st->syn, nm);
    al((void **)&st->words, (size_t)batch * p->n);
    al((void **)&st->conv, st->Bp);
    al((void **)&st->unsat, sizeof(uint32_t) * st->G);
    al((void **)&st->signs, sizeof(uint32_t) * st->G * p->n);
    al((void **)&st->synpack, sizeof(uint32_t) * st->G * p->S * p->z);
    al((void **)&st->active, st->Bp);
    al((void **)&st->gactive, st->G);
    al((void **)&st->take, st->Bp);
    al((void **)&st->iters, st->Bp * sizeof(int64_t));
    al((void **)&st->n_active, sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&st->h_n_active, sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&st->h_flag, 2 * sizeof(int));
    for (int i = 0; i < 2 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&st->ev_flag[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&st->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&st->ev1);
    if (e == cudaSuccess) e = cudaMemsetAsync(st->llr, 0, nl * st->esz, st->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st->stream);
    if (e != cudaSuccess) {
        qcl_state_destroy(st);
        return fail(QCL_ECUDA, "state allocation (B=%lld) failed: %s", (long long)batch, cudaGetErrorString(e));
    }
    *out = st;
    return QCL_OK;
}

int qcl_state_destroy(qcl_state *st) {
    if (!st) return QCL_OK;
    DeviceScope dscope_(st->plan->device);
    if (st->stream) cudaStreamSynchronize(st->stream);
    if (st->fstats) {
        unsigned long long h[16] = {};
        cudaMemcpy(h, st->fstats, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[flow stats] B=%lld W=%d tiles=%llu waited=%llu (%.2f%%) polls=%llu\n", (long long)st->B,
                st->W, h[2], h[0], h[2] ? 100.0 * h[0] / h[2] : 0.0, h[1]);
        const double T = h[2] ? (double)h[2] : 1.0;
        fprintf(stderr, "[flow stats] cycles/tile scheduler: qfree %.0f claim %.0f deps %.0f queue %.0f | consumer: "
                        "full-wait %.0f compute %.0f | storer(x2 tiles): done-wait %.0f issue %.0f read %.0f "
                        "write+release %.0f | loader: ready-wait %.0f empty-wait %.0f issue %.0f\n",
                h[3] / T, h[4] / T, h[5] / T, h[6] / T, h[9] / T, h[10] / T, 2 * h[11] / T, 2 * h[12] / T,
                2 * h[13] / T, 2 * h[14] / T, h[15] / T, h[7] / T, h[8] / T);
    }
    if (st->sweep_exec) cudaGraphExecDestroy(st->sweep_exec);
    if (st->decode_exec) cudaGraphExecDestroy(st->decode_exec);
    for (void *ptr : {st->llr, st->L, st->R, (void *)st->syn, (void *)st->words, (void *)st->conv,
                      (void *)st->unsat, (void *)st->signs, (void *)st->synpack, (void *)st->active, (void *)st->gactive,
                      (void *)st->take, (void *)st->iters,
                      (void *)st->n_active, (void *)st->truths, st->staging, (void *)st->fslot_tab,
                      (void *)st->pframe, (void *)st->piter, (void *)st->pfresh, (void *)st->plane_any,
                      (void *)st->prefill, (void *)st->pcount,
                      (void *)st->fitems, (void *)st->fflags, (void *)st->fcounters, (void *)st->fstats,
                      (void *)st->fitems_et, (void *)st->fsnap, (void *)st->fsign, (void *)st->fet,
                      (void *)st->famask, (void *)st->punits, (void *)st->pbar})
        if (ptr) cudaFree(ptr);
    if (st->h_n_active) cudaFreeHost(st->h_n_active);
    if (st->h_flag) cudaFreeHost(st->h_flag);
    for (int i = 0; i < 2; i++)
        if (st->ev_flag[i]) cudaEventDestroy(st->ev_flag[i]);
    if (st->ev0) cudaEventDestroy(st->ev0);
    if (st->ev1) cudaEventDestroy(st->ev1);
    if (st->staging2) cudaFree(st->staging2);
    st->ring.release();
    if (st->stream) cudaStreamDestroy(st->stream);
    for (int i = 0; i < kSideStreams; i++) {
        if (st->side[i]) cudaStreamDestroy(st->side[i]);
        if (st->join[i]) cudaEventDestroy(st->join[i]);
    }
    if (st->fork) cudaEventDestroy(st->fork);
    delete st;
    return QCL_OK;
}

static int ensure_staging(qcl_state *st, size_t bytes) {
    if (st->staging_bytes >= bytes) return QCL_OK;
    if (st->staging) CK(cudaFree(st->staging));
    st->staging = nullptr;
    st->staging_bytes = 0;
    CK(cudaMalloc(&st->staging, bytes));
    st->staging_bytes = bytes;
    return QCL_OK;
}

static int ensure_staging2(qcl_state *st, size_t bytes) {
    if (st->staging2_bytes >= bytes) return QCL_OK;
    if (st->staging2) CK(cudaFree(st->staging2));
    st->staging2 = nullptr;
    st->staging2_bytes = 0;
    CK(cudaMalloc(&st->staging2, bytes));
    st->staging2_bytes = bytes;
    return QCL_OK;
}

int qcl_state_set_llr(qcl_state *st, const void *llr0, int32_t dtype) {
    if (!st || !llr0) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    const size_t sz = dtype == QCL_DTYPE_F64 ? 8 : 4;
    if (dtype != QCL_DTYPE_F64 && dtype != QCL_DTYPE_F32) return fail(QCL_EVALUE, "unknown llr dtype");
    const size_t bytes = (size_t)st->B * p->n * sz;
    const int64_t total = st->Bp * p->n;
    const unsigned grid = (unsigned)cdiv(total, kBlock);
    if (!host_is_pinned(llr0)) {
        // pageable caller memory (the reference's float64 arrays): convert to the state's
        // type on the host threads while the copy engine moves the previous chunk
        const int64_t cnt = st->B * p->n;
        int rc = ensure_staging(st, (size_t)cnt * st->esz);
        if (rc) return rc;
        if (st->prec == QCL_PREC_FP32) {
            CK(dtype == QCL_DTYPE_F64
                   ? upload_converted(st->ring, (float *)st->staging, (const double *)llr0, cnt, st->stream)
                   : upload_converted(st->ring, (float *)st->staging, (const float *)llr0, cnt, st->stream));
            llr_to_lanes_kernel<float, float><<<grid, kBlock, 0, st->stream>>>(
                (const float *)st->staging, st->B, st->Bp, p->n, st->lw, (float *)st->llr);
        } else {
            CK(dtype == QCL_DTYPE_F64
                   ? upload_converted(st->ring, (double *)st->staging, (const double *)llr0, cnt, st->stream)
                   : upload_converted(st->ring, (double *)st->staging, (const float *)llr0, cnt, st->stream));
            llr_to_lanes_kernel<double, double><<<grid, kBlock, 0, st->stream>>>(
                (const double *)st->staging, st->B, st->Bp, p->n, st->lw, (double *)st->llr);
        }
        CK(cudaGetLastError());
        return QCL_OK;
    }
    int rc = ensure_staging(st, bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(st->staging, llr0, bytes, cudaMemcpyHostToDevice, st->stream));
    if (st->prec == QCL_PREC_FP32) {
        if (dtype == QCL_DTYPE_F64)
            llr_to_lanes_kernel<float, double><<<grid, kBlock, 0, st->stream>>>(
                (const double *)st->staging, st->B, st->Bp, p->n, st->lw, (float *)st->llr);
        else
            llr_to_lanes_kernel<float, float><<<grid, kBlock, 0, st->stream>>>(
                (const float *)st->staging, st->B, st->Bp, p->n, st->lw, (float *)st->llr);
    } else {
        if (dtype == QCL_DTYPE_F64)
            llr_to_lanes_kernel<double, double><<<grid, kBlock, 0, st->stream>>>(
                (const double *)st->staging, st->B, st->Bp, p->n, st->lw, (double *)st->llr);
        else
            llr_to_lanes_kernel<double, float><<<grid, kBlock, 0, st->stream>>>(
                (const float *)st->staging, st->B, st->Bp, p->n, st->lw, (double *)st->llr);
    }
    CK(cudaGetLastError());
    return QCL_OK;
}

int qcl_state_set_llr_synthetic(qcl_state *st, uint64_t seed, int64_t snr_idx, int64_t first_frame, double snr,
                                int32_t encode_mode) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    if (!(snr > 0)) return fail(QCL_EVALUE, "snr must be positive");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    if (encode_mode && !st->truths) CK(cudaMalloc(&st->truths, (size_t)st->B * p->n));
    const double sigma2 = 1.0 / snr, sigma = sqrt(sigma2);
    const int64_t total = st->Bp * cdiv(p->n, 4);
    const unsigned grid = (unsigned)cdiv(total, kBlock);
    uint8_t *tr = encode_mode ? st->truths : nullptr;
    if (st->prec == QCL_PREC_FP32)
        synth_llr_kernel<float><<<grid, kBlock, 0, st->stream>>>(st->B, st->Bp, p->n, st->lw, seed,
                                                                  (uint32_t)snr_idx, first_frame, sigma, sigma2,
                                                                  encode_mode, (float *)st->llr, tr);
    else
        synth_llr_kernel<double><<<grid, kBlock, 0, st->stream>>>(st->B, st->Bp, p->n, st->lw, seed,
                                                                   (uint32_t)snr_idx, first_frame, sigma, sigma2,
                                                                   encode_mode, (double *)st->llr, tr);
    CK(cudaGetLastError());
    st->truths_valid = encode_mode != 0;
    if (encode_mode) {
        SlotRange r = slot_range(st, 0, p->S, 1);
        dim3 g2((unsigned)((int64_t)st->G * p->S * r.bps));
        syndrome_of_words_kernel<<<g2, kBlock, 0, st->stream>>>(r, st->truths, st->B, st->syn);
        CK(cudaGetLastError());
        st->has_syn = true;
        int rc = enqueue_syn_pack(st);
        if (rc) return rc;
    } else {
        st->has_syn = false;
    }
    return QCL_OK;
}

int qcl_state_truths(qcl_state *st, uint8_t *words) {
    if (!st || !words) return fail(QCL_EVALUE, "NULL argument");
    DEVICE_SCOPE(st->plan->device);
    if (!st->truths || !st->truths_valid) {
        CK(cudaStreamSynchronize(st->stream));
        memset(words, 0, (size_t)st->B * st->plan->n);
        return QCL_OK;
    }
    CK(cudaMemcpyAsync(words, st->truths, (size_t)st->B * st->plan->n, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_frame_errors(qcl_state *st, uint8_t *mismatch) {
    if (!st || !mismatch) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    CK(cudaMemsetAsync(st->take, 0, st->B, st->stream));  // reused as the per-frame flag buffer
    const int64_t units = (p->n % 16 == 0) ? p->n / 16 : p->n;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(units, kBlock), 64));
    frame_mismatch_kernel<<<dim3(gx, (unsigned)std::min<int64_t>(st->B, 65535)), kBlock, 0, st->stream>>>(
        st->words, st->truths_valid ? st->truths : nullptr, p->n, st->B, st->take);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(mismatch, st->take, st->B, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_get_llr(qcl_state *st, double *llr) {
    if (!st || !llr) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    int rc = ensure_staging(st, (size_t)st->B * p->n * 8);
    if (rc) return rc;
    const int64_t total = st->B * p->n;
    const unsigned grid = (unsigned)cdiv(total, kBlock);
    if (st->prec == QCL_PREC_FP32)
        state_out_kernel<float, float><<<grid, kBlock, 0, st->stream>>>((const float *)st->llr, nullptr, st->B, p->n, 0,
                                                                  st->lw, (double *)st->staging, nullptr);
    else
        state_out_kernel<double, double><<<grid, kBlock, 0, st->stream>>>((const double *)st->llr, nullptr, st->B, p->n,
                                                                   0, st->lw, (double *)st->staging, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(llr, st->staging, total * 8, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_set_syndrome(qcl_state *st, const uint8_t *syndrome) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    if (!syndrome) {
        st->has_syn = false;
        return QCL_OK;
    }
    const size_t bytes = (size_t)st->B * p->m;
    // an all-zero target (the campaign default, bench.py:227-228) is detected on the host
    // and never uploaded: it takes the syndrome-free kernel variant, which does not read
    // the per-check syndrome bytes at all
    if (!host_any_nonzero(syndrome, (int64_t)bytes)) {
        st->has_syn = false;
        return QCL_OK;
    }
    int rc = ensure_staging(st, bytes);
    if (rc) return rc;
    if (host_is_pinned(syndrome))
        CK(cudaMemcpyAsync(st->staging, syndrome, bytes, cudaMemcpyHostToDevice, st->stream));
    else
        CK(upload_converted(st->ring, (uint8_t *)st->staging, syndrome, (int64_t)bytes, st->stream));
    CK(cudaMemsetAsync(st->n_active, 0, sizeof(int), st->stream));
    const int64_t total = st->Bp * p->m;
    syndrome_to_lanes_kernel<<<(unsigned)cdiv(total, kBlock), kBlock, 0, st->stream>>>(
        (const uint8_t *)st->staging, p->slots, st->B, st->Bp, p->S, p->z, st->lw, st->syn, st->n_active);
    CK(cudaGetLastError());
    st->has_syn = true;
    return enqueue_syn_pack(st);
}

// new_state (decoder.py:191-202): L = clip(llr), R = 0.  zero_r = false when the first
// flow sweep treats every message as zero itself (FlowArgs::fresh_t): saves writing R
// (964 MB at 64 codewords) before every decode.
static int enqueue_reset(qcl_state *st, double clip, bool zero_r = true) {
    const qcl_plan *p = st->plan;
    const int64_t nl = st->Bp * p->n;
    if (st->prec == QCL_PREC_FP32)  // 4 values per thread when nl % 4 == 0
        reset_kernel<float><<<(unsigned)cdiv(nl % 4 == 0 ? nl / 4 : nl, kBlock), kBlock, 0, st->stream>>>(
            (const float *)st->llr, (float *)st->L, nl, clip);
    else
        reset_kernel<double><<<(unsigned)cdiv(nl, kBlock), kBlock, 0, st->stream>>>((const double *)st->llr,
                                                                                     (double *)st->L, nl, clip);
    CK(cudaGetLastError());
    if (zero_r) CK(cudaMemsetAsync(st->R, 0, (size_t)st->Bp * p->E * p->z * st->resz, st->stream));
    st->launches_all++;
    return QCL_OK;
}

int qcl_state_reset(qcl_state *st, double llr_clip) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    if (!(llr_clip > 0)) return fail(QCL_EVALUE, "llr_clip must be positive");
    DEVICE_SCOPE(st->plan->device);
    return enqueue_reset(st, llr_clip);
}

int qcl_state_upload(qcl_state *st, const double *posterior, const double *messages) {
    if (!st || !posterior) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    const int64_t Ez = (int64_t)p->E * p->z;
    const size_t pb = (size_t)st->B * p->n * 8, mb = (size_t)st->B * Ez * 8;
    int rc = ensure_staging(st, pb + mb);
    if (rc) return rc;
    double *sp = (double *)st->staging, *sm = sp + st->B * p->n;
    CK(cudaMemcpyAsync(sp, posterior, pb, cudaMemcpyHostToDevice, st->stream));
    if (messages) CK(cudaMemcpyAsync(sm, messages, mb, cudaMemcpyHostToDevice, st->stream));
    const int64_t total = st->Bp * std::max<int64_t>(p->n, Ez);
    const unsigned grid = (unsigned)cdiv(total, kBlock);
    if (st->msg16)
        state_in_kernel<float, __half><<<grid, kBlock, 0, st->stream>>>(sp, messages ? sm : nullptr, st->B, p->n,
                                                                         Ez, st->lw, (float *)st->L, (__half *)st->R,
                                                                         st->Bp);
    else if (st->prec == QCL_PREC_FP32)
        state_in_kernel<float><<<grid, kBlock, 0, st->stream>>>(sp, messages ? sm : nullptr, st->B, p->n, Ez,
                                                                 st->lw, (float *)st->L, (float *)st->R, st->Bp);
    else
        state_in_kernel<double><<<grid, kBlock, 0, st->stream>>>(sp, messages ? sm : nullptr, st->B, p->n, Ez,
                                                                  st->lw, (double *)st->L, (double *)st->R, st->Bp);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_download(qcl_state *st, double *posterior, double *messages) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    const int64_t Ez = (int64_t)p->E * p->z;
    const size_t pb = (size_t)st->B * p->n * 8, mb = (size_t)st->B * Ez * 8;
    int rc = ensure_staging(st, pb + mb);
    if (rc) return rc;
    double *sp = (double *)st->staging, *sm = sp + st->B * p->n;
    const int64_t total = st->B * std::max<int64_t>(p->n, Ez);
    const unsigned grid = (unsigned)cdiv(total, kBlock);
    if (st->msg16)
        state_out_kernel<float, __half><<<grid, kBlock, 0, st->stream>>>((const float *)st->L, (const __half *)st->R,
                                                                          st->B, p->n, Ez, st->lw, sp, sm);
    else if (st->prec == QCL_PREC_FP32)
        state_out_kernel<float><<<grid, kBlock, 0, st->stream>>>((const float *)st->L, (const float *)st->R, st->B,
                                                                  p->n, Ez, st->lw, sp, sm);
    else
        state_out_kernel<double><<<grid, kBlock, 0, st->stream>>>((const double *)st->L, (const double *)st->R,
                                                                   st->B, p->n, Ez, st->lw, sp, sm);
    CK(cudaGetLastError());
    if (posterior) CK(cudaMemcpyAsync(posterior, sp, pb, cudaMemcpyDeviceToHost, st->stream));
    if (messages) CK(cudaMemcpyAsync(messages, sm, mb, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_layers(qcl_state *st, int32_t first, int32_t count, double llr_clip, double phi_epsilon) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    if (first < 0 || count < 0 || first + count > p->n_layers)
        return fail(QCL_EVALUE, "layer range [%d, %d) outside [0, %d)", first, first + count, p->n_layers);
    DEVICE_SCOPE(p->device);
    if (st->msg16) {
        if (!use_flow(st) || first != 0 || count != p->n_layers) return msg16_unsupported(st, "whole sweeps only");
        int rc = ensure_flow(st, 1);
        if (rc) return rc;
        if (!use_flow(st)) return msg16_unsupported(st, "tables exceed shared memory");
    }
    const bool saved_et = st->g_et;
    st->g_et = false;  // direct layer launches never skip
    if (use_flow(st) && first == 0 && count == p->n_layers) {
        int rc = ensure_flow(st, 1);
        if (rc) {
            st->g_et = saved_et;
            return rc;
        }
    }
    if (use_flow(st) && first == 0 && count == p->n_layers) {  // one whole sweep: flow engine
        int rc = enqueue_flow_reset(st, 1);
        if (!rc) rc = enqueue_flow(st, llr_clip, phi_epsilon, 0, 1, 0, false);
        st->g_et = saved_et;
        if (rc) return rc;
        CK(cudaStreamSynchronize(st->stream));
        return QCL_OK;
    }
    for (int l = first; l < first + count; l++) enqueue_layer(st, l, llr_clip, phi_epsilon, st->stream, 0, st->G, true);
    st->g_et = saved_et;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_hard_decision(qcl_state *st, uint8_t *words) {
    if (!st || !words) return fail(QCL_EVALUE, "NULL argument");
    DEVICE_SCOPE(st->plan->device);
    int rc = enqueue_signs(st);
    if (!rc) rc = enqueue_words(st, nullptr);
    if (rc) return rc;
    CK(cudaMemcpyAsync(words, st->words, (size_t)st->B * st->plan->n, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_syndrome_ok(qcl_state *st, uint8_t *ok) {
    if (!st || !ok) return fail(QCL_EVALUE, "NULL argument");
    DEVICE_SCOPE(st->plan->device);
    int rc = enqueue_check(st);
    if (rc) return rc;
    std::vector<uint32_t> un(st->G);
    CK(cudaMemcpyAsync(un.data(), st->unsat, sizeof(uint32_t) * st->G, cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    for (int64_t b = 0; b < st->B; b++) ok[b] = !((un[b >> st->lw] >> (b & (st->W - 1))) & 1u);
    return QCL_OK;
}

static int validate_cfg(const qcl_config *cfg) {
    if (!cfg) return fail(QCL_EVALUE, "config is NULL");
    if (cfg->max_iterations < 1) return fail(QCL_EVALUE, "max_iterations must be at least 1");
    if (!(cfg->llr_clip > 0)) return fail(QCL_EVALUE, "llr_clip must be positive");
    if (!(cfg->phi_epsilon > 0 && cfg->phi_epsilon < 1)) return fail(QCL_EVALUE, "phi_epsilon must be in (0, 1)");
    if (cfg->precision != QCL_PREC_FP32 && cfg->precision != QCL_PREC_FP64 && cfg->precision != QCL_PREC_FP32_MSG16)
        return fail(QCL_EVALUE, "unknown precision %d", cfg->precision);
    return QCL_OK;
}

// Enqueue a full decode (decoder.py:275-312) on the state's stream.  With `sync` the
// early-termination loop stops as soon as every frame has converged, reading the
// device's active count one iteration behind (the sweep after convergence is already
// queued, which changes nothing: converged frames are frozen).  Without `sync` nothing
// waits on the host: after the last frame converges the remaining layer launches
// return immediately (they read the device count), so results are identical.
// The decode body without host synchronisation: init, reset, the sweeps (and per-sweep
// early-termination bookkeeping), final check and words.  Captured once into a
// whole-decode graph; the only host work per decode is then one graph launch.
// Early-termination decode on the flow engine with the per-sweep check fused into the one
// launch (flow.cuh, "Fused early termination"): init, reset, flags/counters, the launch
// (CUDA events around it when profiling), words.
static int enqueue_decode_fused_et(qcl_state *st, const qcl_config *cfg) {
    int rc;
    const qcl_plan *p = st->plan;
    decode_init_kernel<<<(unsigned)cdiv(st->Bp, kBlock), kBlock, 0, st->stream>>>(
        st->B, st->Bp, cfg->max_iterations, st->active, st->conv, st->iters, st->n_active);
    enqueue_group_active(st);
    amask_init_kernel<<<(unsigned)cdiv(st->G, kBlock), kBlock, 0, st->stream>>>(st->G, st->lw, st->B, st->famask);
    st->launches_all += 2;
    st->g_et = true;
    if ((rc = enqueue_reset(st, cfg->llr_clip, false))) return rc;  // sweep 0 zeroes r_old itself
    if (p->n_untouched) {  // columns without edges: no tile writes their snapshot; L never changes
        const int64_t total = (int64_t)st->G * p->n_untouched * p->z;
        snap_untouched_kernel<<<(unsigned)cdiv(total, kBlock), kBlock, 0, st->stream>>>(
            (const float *)st->L, p->funtouched, p->n_untouched, p->z, p->n, st->G, st->lw, st->fsnap);
        st->launches_all++;
    }
    if ((rc = enqueue_flow_reset(st, 1))) return rc;
    CK(cudaMemsetAsync(st->fet, 0, sizeof(int) * 5 * QCL_FLAG_STRIDE * (size_t)st->G, st->stream));
    cudaEvent_t a = nullptr, b = nullptr;
    if (st->profiling) {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st->stream));
    }
    // degree-1 deferral as in the no-ET decode: the snapshots take the true posteriors; a
    // decode that stops early leaves the degree-1 columns' L slots holding the next sweep's
    // q (only qcl_state_download sees that; words, flags and iterations do not)
    if ((rc = enqueue_flow(st, cfg->llr_clip, cfg->phi_epsilon, 0, cfg->max_iterations, 0, true,
                           flow_defer_last(cfg->max_iterations), nullptr, 0, true)))
        return rc;
    if (st->profiling) {
        CK(cudaEventRecord(b, st->stream));
        st->sweep_events.push_back({a, b});
    }
    const uint8_t *snap_last = st->fsnap + (size_t)((cfg->max_iterations - 1) & 1) * st->G * p->n;
    et_words_kernel<<<(unsigned)cdiv(p->n, kBlock), kBlock, 0, st->stream>>>(snap_last, st->fsign, st->conv, p->n,
                                                                              st->lw, st->B, st->words);
    st->launches_all++;
    CK(cudaGetLastError());
    return QCL_OK;
}

static int enqueue_decode_body(qcl_state *st, const qcl_config *cfg) {
    int rc;
    const unsigned gb = (unsigned)cdiv(st->B, kBlock);
    const bool et = cfg->early_termination != 0;
    if (et && st->fused_et) return enqueue_decode_fused_et(st, cfg);
    decode_init_kernel<<<(unsigned)cdiv(st->Bp, kBlock), kBlock, 0, st->stream>>>(
        st->B, st->Bp, cfg->max_iterations, st->active, st->conv, st->iters, st->n_active);
    st->launches_all++;
    enqueue_group_active(st);
    st->g_et = et;
    const bool flow = st->flow_decode;
    const bool persist = st->persist_decode;
    if ((rc = enqueue_reset(st, cfg->llr_clip, !flow))) return rc;  // flow: sweep 0 zeroes r_old itself
    if (persist && !et) {  // every sweep in one cooperative launch
        if ((rc = enqueue_persist(st, cfg->max_iterations, false))) return rc;
    }
    if (flow) {
        if ((rc = enqueue_flow_reset(st, et ? cfg->max_iterations : 1))) return rc;
        if (!et) {  // every sweep in one persistent launch, degree-1 edges deferred
            if ((rc = enqueue_flow(st, cfg->llr_clip, cfg->phi_epsilon, 0, cfg->max_iterations, 0, false,
                                   flow_defer_last(cfg->max_iterations), nullptr, 0)))
                return rc;
        }
    }
    for (int t = 1; t <= cfg->max_iterations; t++) {
        if ((flow || persist) && !et) break;
        const int64_t before = st->launches_layer;
        if (persist) {
            if ((rc = enqueue_persist(st, 1, true))) return rc;
            st->launches_all -= st->launches_layer - before;  // counted below
        } else if (flow) {
            if ((rc = enqueue_flow(st, cfg->llr_clip, cfg->phi_epsilon, t - 1, 1, t - 1, true, -1, nullptr, 0)))
                return rc;
            st->launches_all -= st->launches_layer - before;  // counted below
        } else {
            enqueue_sweep(st, cfg->llr_clip, cfg->phi_epsilon);
        }
        st->launches_all += st->launches_layer - before;
        if (!et) continue;
        if ((rc = enqueue_check(st, st->gactive))) return rc;
        et_update_kernel<<<gb, kBlock, 0, st->stream>>>(st->B, t, st->unsat, st->lw, st->active, st->take, st->conv,
                                                        st->iters, st->n_active);
        st->launches_all++;
        if ((rc = enqueue_words(st, st->take))) return rc;
        enqueue_group_active(st);
    }
    if ((rc = enqueue_check(st, st->gactive))) return rc;
    finalize_kernel<<<gb, kBlock, 0, st->stream>>>(st->B, st->unsat, st->lw, st->active, st->take, st->conv);
    st->launches_all++;
    return enqueue_words(st, st->take);
}

// Enqueue a full decode (decoder.py:275-312) on the state's stream.
//  * default: one launch of the whole-decode graph (rebuilt when the config, the
//    syndrome presence or the engine changes).  With early termination, every layer
//    launch after the last convergence returns at once (it reads the device count), so
//    results equal the reference's early break: converged frames are frozen.
//  * sync && early termination: the sweep graph per iteration, and the host stops once
//    every frame converged (active count read one iteration behind).
//  * profiling: the sweep graph per iteration with CUDA events around each sweep.
static int enqueue_decode(qcl_state *st, const qcl_config *cfg, bool sync) {
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (cfg->precision != st->api_prec) return fail(QCL_EVALUE, "config precision differs from the state's");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    st->launches_layer = st->launches_all = 0;
    st->layer_ms = 0;
    const bool et = cfg->early_termination != 0;
    if (use_flow(st) && (rc = ensure_flow(st, cfg->max_iterations))) return rc;  // allocations outside capture
    st->flow_decode = use_flow(st) && (int64_t)cfg->max_iterations * st->f_sweep_items * st->f_nblk + 8LL * st->f_grid <
                                           (1LL << 31);
    if (st->msg16 && !st->flow_decode) return msg16_unsupported(st, "this decode");
    bool fused = false;
    if (et && st->flow_decode && use_flow_et(st)) {
        if ((rc = ensure_flow_et(st))) return rc;
        fused = (int64_t)cfg->max_iterations * st->f_sweep_items_et * st->f_nblk + 8LL * st->f_grid < (1LL << 31);
    }
    st->fused_et = fused;
    st->persist_decode = !st->flow_decode && use_persist(st);
    if (st->persist_decode && (rc = ensure_persist(st, cfg->llr_clip, cfg->phi_epsilon))) return rc;
    if (fused && st->profiling) {
        CK(cudaEventRecord(st->ev0, st->stream));
        if ((rc = enqueue_decode_fused_et(st, cfg))) return rc;
        CK(cudaEventRecord(st->ev1, st->stream));
        return QCL_OK;
    }
    if (!st->profiling && !(sync && et && !fused)) {
        const bool stale = !st->decode_exec || st->d_clip != cfg->llr_clip || st->d_eps != cfg->phi_epsilon ||
                           st->d_syn != st->has_syn || st->d_et != et || st->d_iters != cfg->max_iterations ||
                           st->d_engine != st->engine;
        if (stale) {
            if (st->decode_exec) cudaGraphExecDestroy(st->decode_exec);
            st->decode_exec = nullptr;
            cudaGraph_t graph;
            CK(cudaStreamBeginCapture(st->stream, cudaStreamCaptureModeThreadLocal));
            rc = enqueue_decode_body(st, cfg);
            cudaError_t e = cudaStreamEndCapture(st->stream, &graph);
            if (rc) return rc;
            CK(e);
            e = cudaGraphInstantiate(&st->decode_exec, graph, 0);
            cudaGraphDestroy(graph);
            CK(e);
            st->d_clip = cfg->llr_clip;
            st->d_eps = cfg->phi_epsilon;
            st->d_syn = st->has_syn;
            st->d_et = et;
            st->d_iters = cfg->max_iterations;
            st->d_engine = st->engine;
            st->d_launches_layer = st->launches_layer;
            st->d_launches_all = st->launches_all;
        }
        st->launches_layer = st->d_launches_layer;
        st->launches_all = st->d_launches_all;
        CK(cudaEventRecord(st->ev0, st->stream));
        CK(cudaGraphLaunch(st->decode_exec, st->stream));
        CK(cudaEventRecord(st->ev1, st->stream));
        CK(cudaGetLastError());
        return QCL_OK;
    }
    CK(cudaEventRecord(st->ev0, st->stream));
    decode_init_kernel<<<(unsigned)cdiv(st->Bp, kBlock), kBlock, 0, st->stream>>>(
        st->B, st->Bp, cfg->max_iterations, st->active, st->conv, st->iters, st->n_active);
    st->launches_all++;
    enqueue_group_active(st);
    const unsigned gb = (unsigned)cdiv(st->B, kBlock);
    const bool flow = st->flow_decode;
    if ((rc = enqueue_reset(st, cfg->llr_clip, !flow))) return rc;  // flow: sweep 0 zeroes r_old itself
    if (flow && (rc = enqueue_flow_reset(st, cfg->max_iterations))) return rc;
    for (int t = 1; t <= cfg->max_iterations; t++) {
        if (flow) {
            // no early termination: all sweeps in one launch (timed as one "sweep" unit)
            const int T = et ? 1 : cfg->max_iterations;
            cudaEvent_t a = nullptr, b = nullptr;
            if (st->profiling) {
                CK(cudaEventCreate(&a));
                CK(cudaEventCreate(&b));
                CK(cudaEventRecord(a, st->stream));
            }
            if ((rc = enqueue_flow(st, cfg->llr_clip, cfg->phi_epsilon, t - 1, T, t - 1, et,
                                   et ? -1 : flow_defer_last(cfg->max_iterations), nullptr, 0)))
                return rc;
            if (st->profiling) {
                CK(cudaEventRecord(b, st->stream));
                st->sweep_events.push_back({a, b});
            }
            if (!et) break;
        } else if ((rc = run_sweep(st, cfg->llr_clip, cfg->phi_epsilon, et))) {
            return rc;
        }
        if (!et) continue;
        if ((rc = enqueue_check(st, st->gactive))) return rc;
        et_update_kernel<<<gb, kBlock, 0, st->stream>>>(st->B, t, st->unsat, st->lw, st->active, st->take, st->conv,
                                                        st->iters, st->n_active);
        st->launches_all++;
        if ((rc = enqueue_words(st, st->take))) return rc;
        enqueue_group_active(st);
        if (!sync) continue;
        CK(cudaMemcpyAsync(st->h_flag + (t & 1), st->n_active, sizeof(int), cudaMemcpyDeviceToHost, st->stream));
        CK(cudaEventRecord(st->ev_flag[t & 1], st->stream));
        if (t >= 2) {
            CK(cudaEventSynchronize(st->ev_flag[(t - 1) & 1]));
            if (st->h_flag[(t - 1) & 1] == 0) break;
        }
    }
    if ((rc = enqueue_check(st, st->gactive))) return rc;
    finalize_kernel<<<gb, kBlock, 0, st->stream>>>(st->B, st->unsat, st->lw, st->active, st->take, st->conv);
    st->launches_all++;
    if ((rc = enqueue_words(st, st->take))) return rc;
    CK(cudaEventRecord(st->ev1, st->stream));
    CK(cudaGetLastError());
    return QCL_OK;
}

static int finish_decode(qcl_state *st, float *elapsed_ms) {
    CK(cudaEventSynchronize(st->ev1));
    CK(cudaGetLastError());
    if (elapsed_ms) {
        // a wait with no decode recorded yet (only uploads or downloads queued): 0 ms
        const cudaError_t e = cudaEventElapsedTime(elapsed_ms, st->ev0, st->ev1);
        if (e == cudaErrorInvalidResourceHandle) {
            cudaGetLastError();
            *elapsed_ms = 0.0f;
        } else {
            CK(e);
        }
    }
    for (auto &ev : st->sweep_events) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev.first, ev.second));
        st->layer_ms += ms;
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    st->sweep_events.clear();
    return QCL_OK;
}

int qcl_state_decode(qcl_state *st, const qcl_config *cfg, float *elapsed_ms) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    int rc = enqueue_decode(st, cfg, true);
    if (rc) return rc;
    return finish_decode(st, elapsed_ms);
}

static int sms_of(const qcl_state *st) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st->plan->device);
    return sms;
}

// Frame pool: n_frames device-generated frames (all-zero word, zero syndrome) streamed
// through the state's lanes with early termination (kernels.cuh, "frame pool").  Outcomes
// land at their frame index: conv, iters, err (frame error as bench.py:236-237).
int qcl_state_decode_pool(qcl_state *st, const qcl_config *cfg, uint64_t seed, int64_t snr_idx, int64_t first_frame,
                          int64_t n_frames, double snr, uint8_t *conv, int64_t *iters, uint8_t *err,
                          float *elapsed_ms) {
    if (!st || !conv || !iters || !err) return fail(QCL_EVALUE, "NULL argument");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (cfg->precision != st->api_prec) return fail(QCL_EVALUE, "config precision differs from the state's");
    if (!cfg->early_termination) return fail(QCL_EVALUE, "the frame pool needs early termination");
    if (n_frames < 1) return fail(QCL_EVALUE, "n_frames must be at least 1");
    if (!(snr > 0)) return fail(QCL_EVALUE, "snr must be positive");
    if (!use_flow(st)) return fail(QCL_EUNSUP, "the frame pool runs on the flow engine (FP32, engine 4)");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    if ((rc = ensure_flow(st, 2))) return rc;
    if (!use_flow(st)) return fail(QCL_EUNSUP, "the frame pool runs on the flow engine (FP32, engine 4)");
    auto al = [&](void **ptr, size_t bytes) -> int {
        if (*ptr) return QCL_OK;
        CK(cudaMalloc(ptr, std::max<size_t>(bytes, 16)));
        return QCL_OK;
    };
    if ((rc = al((void **)&st->pframe, sizeof(int64_t) * st->Bp)) || (rc = al((void **)&st->piter, 4 * st->Bp)) ||
        (rc = al((void **)&st->pfresh, 4 * st->G)) || (rc = al((void **)&st->plane_any, 4 * st->G)) ||
        (rc = al((void **)&st->prefill, 4 * st->Bp)) || (rc = al((void **)&st->pcount, 16)))
        return rc;
    uint8_t *d_conv = nullptr, *d_err = nullptr;
    int64_t *d_iters = nullptr;
    CK(cudaMalloc(&d_conv, n_frames));
    CK(cudaMalloc(&d_err, n_frames));
    CK(cudaMalloc(&d_iters, 8 * n_frames));
    cudaStream_t sm = st->stream;
    const double sigma2 = 1.0 / snr, sigma = sqrt(sigma2);
    // the first frames fill the lanes: lanes [0, first) get frames first_frame.. in order
    const int64_t first = std::min<int64_t>(st->B, n_frames);
    std::vector<int64_t> h_frame(st->Bp, -1);
    std::vector<uint8_t> h_active(st->Bp, 0);
    for (int64_t b = 0; b < first; b++) {
        h_frame[b] = first_frame + b;
        h_active[b] = 1;
    }
    const int32_t h_count[3] = {0, (int32_t)first, 0};  // refills, frames handed out, sweep
    const int h_n_active = (int)first;
    CK(cudaMemcpyAsync(st->pframe, h_frame.data(), 8 * st->Bp, cudaMemcpyHostToDevice, sm));
    CK(cudaMemcpyAsync(st->active, h_active.data(), st->Bp, cudaMemcpyHostToDevice, sm));
    CK(cudaMemcpyAsync(st->pcount, h_count, 12, cudaMemcpyHostToDevice, sm));
    CK(cudaMemcpyAsync(st->n_active, &h_n_active, sizeof(int), cudaMemcpyHostToDevice, sm));
    CK(cudaMemsetAsync(st->piter, 0, 4 * st->Bp, sm));
    CK(cudaMemsetAsync(st->pfresh, 0, 4 * st->G, sm));
    CK(cudaStreamSynchronize(sm));  // the pageable sources above
    if ((rc = qcl_state_set_llr_synthetic(st, seed, snr_idx, first_frame, snr, 0))) return rc;
    st->has_syn = false;
    st->pool_active = true;
    st->g_et = true;
    const unsigned gb = (unsigned)cdiv(st->Bp, kBlock);
    const unsigned qgrid = (unsigned)cdiv((p->n + 3) / 4, kBlock);
    // every frame needs at most max_iterations sweeps and the lanes work concurrently
    const int64_t max_sweeps = (int64_t)cfg->max_iterations * (cdiv(n_frames, st->B) + 1) + 1;
    // Sweeps run as a CUDA graph of kPoolChunk sweeps: the sweep index lives in device memory
    // (pcount[2], advanced by pool_update with the claim counter reset), so every sweep has the
    // same launch parameters and the host only launches chunks and reads the active count one
    // chunk behind.  Sweeps after the last lane retired cost ~nothing (the flow launch returns
    // at once, the bookkeeping kernels find no active lane).
    constexpr int kPoolChunk = 4;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CK(cudaStreamBeginCapture(sm, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < kPoolChunk && !rc; k++) {
        if ((rc = enqueue_flow(st, cfg->llr_clip, cfg->phi_epsilon, 0, 1, 0, true, -1, st->pcount + 2, 0))) break;
        cudaMemsetAsync(st->pfresh, 0, 4 * st->G, sm);
        if ((rc = enqueue_check(st, st->gactive))) break;
        cudaMemsetAsync(st->plane_any, 0, 4 * st->G, sm);
        lane_any_kernel<<<(unsigned)(2 * sms_of(st)), kBlock, 0, sm>>>(st->signs, p->n, st->G, st->gactive,
                                                                      st->plane_any);
        cudaMemsetAsync(st->pcount, 0, sizeof(int32_t), sm);
        pool_update_kernel<<<gb, kBlock, 0, sm>>>(st->Bp, st->lw, cfg->max_iterations, st->unsat, st->plane_any,
                                                 first_frame, n_frames, st->pframe, st->piter, st->active,
                                                 st->n_active, d_conv, d_iters, d_err, st->pcount, st->prefill,
                                                 st->pfresh, st->fcounters);
        pool_refill_kernel<<<dim3(qgrid, (unsigned)std::min<int64_t>(st->Bp, 8)), kBlock, 0, sm>>>(
            st->pcount, st->prefill, st->pframe, p->n, st->lw, seed, (uint32_t)snr_idx, sigma, sigma2,
            cfg->llr_clip, (float *)st->llr, (float *)st->L);
        enqueue_group_active(st);
    }
    cudaError_t ce = cudaStreamEndCapture(sm, &graph);
    if (!rc && ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (!rc && ce != cudaSuccess) rc = fail(QCL_ECUDA, "pool sweep graph: %s", cudaGetErrorString(ce));
    if (rc) {
        if (exec) cudaGraphExecDestroy(exec);
        cudaFree(d_conv);
        cudaFree(d_err);
        cudaFree(d_iters);
        st->pool_active = false;
        return rc;
    }
    // the timed region starts here (graph capture and instantiation are host set-up)
    CK(cudaEventRecord(st->ev0, sm));
    if ((rc = enqueue_reset(st, cfg->llr_clip, false))) return rc;  // sweep 0 zeroes r_old itself
    enqueue_group_active(st);
    CK(cudaMemsetAsync(st->fflags, 0, sizeof(int) * QCL_FLAG_STRIDE * (size_t)st->G * st->f_nkb_total, sm));
    CK(cudaMemsetAsync(st->fcounters, 0, sizeof(int), sm));
    for (int64_t c = 0; !rc && c * kPoolChunk < max_sweeps; c++) {
        cudaError_t e = cudaGraphLaunch(exec, sm);
        // stop once every lane retired: the active count is read one chunk behind
        if (e == cudaSuccess) e = cudaMemcpyAsync(st->h_flag + (c & 1), st->n_active, sizeof(int), cudaMemcpyDeviceToHost, sm);
        if (e == cudaSuccess) e = cudaEventRecord(st->ev_flag[c & 1], sm);
        if (e == cudaSuccess && c >= 1) e = cudaEventSynchronize(st->ev_flag[(c - 1) & 1]);
        if (e != cudaSuccess) {
            rc = fail(QCL_ECUDA, "pool sweep: %s", cudaGetErrorString(e));
            break;
        }
        if (c >= 1 && st->h_flag[(c - 1) & 1] == 0) break;
    }
    if (exec) cudaGraphExecDestroy(exec);
    st->pool_active = false;
    CK(cudaEventRecord(st->ev1, sm));
    if (!rc) {
        CK(cudaMemcpyAsync(conv, d_conv, n_frames, cudaMemcpyDeviceToHost, sm));
        CK(cudaMemcpyAsync(err, d_err, n_frames, cudaMemcpyDeviceToHost, sm));
        CK(cudaMemcpyAsync(iters, d_iters, 8 * n_frames, cudaMemcpyDeviceToHost, sm));
    }
    cudaError_t e = cudaStreamSynchronize(sm);
    if (elapsed_ms && e == cudaSuccess) cudaEventElapsedTime(elapsed_ms, st->ev0, st->ev1);
    cudaFree(d_conv);
    cudaFree(d_err);
    cudaFree(d_iters);
    if (rc) return rc;
    CK(e);
    return QCL_OK;
}

int qcl_state_decode_async(qcl_state *st, const qcl_config *cfg) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    return enqueue_decode(st, cfg, false);
}

int qcl_state_results_async(qcl_state *st, uint8_t *words, uint8_t *converged, int64_t *iterations) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    if (words) CK(cudaMemcpyAsync(words, st->words, (size_t)st->B * p->n, cudaMemcpyDeviceToHost, st->stream));
    if (converged) CK(cudaMemcpyAsync(converged, st->conv, st->B, cudaMemcpyDeviceToHost, st->stream));
    if (iterations)
        CK(cudaMemcpyAsync(iterations, st->iters, st->B * sizeof(int64_t), cudaMemcpyDeviceToHost, st->stream));
    return QCL_OK;
}

int qcl_state_wait(qcl_state *st, float *decode_ms) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    DEVICE_SCOPE(st->plan->device);
    CK(cudaStreamSynchronize(st->stream));  // everything queued on the state, results included
    return finish_decode(st, decode_ms);
}

int qcl_state_set_syndrome_hint(qcl_state *st, const uint8_t *syndrome, int32_t nonzero) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    const size_t bytes = (size_t)st->B * p->m;
    // nonzero < 0: the caller did not look; the host threads check for an all-zero target
    if (syndrome && nonzero < 0) nonzero = host_any_nonzero(syndrome, (int64_t)bytes);
    if (!syndrome || !nonzero) {
        st->has_syn = false;
        return QCL_OK;
    }
    int rc = ensure_staging2(st, bytes);
    if (rc) return rc;
    if (host_is_pinned(syndrome))
        CK(cudaMemcpyAsync(st->staging2, syndrome, bytes, cudaMemcpyHostToDevice, st->stream));
    else
        CK(upload_converted(st->ring, (uint8_t *)st->staging2, syndrome, (int64_t)bytes, st->stream));
    const int64_t total = st->Bp * p->m;
    syndrome_to_lanes_kernel<<<(unsigned)cdiv(total, kBlock), kBlock, 0, st->stream>>>(
        (const uint8_t *)st->staging2, p->slots, st->B, st->Bp, p->S, p->z, st->lw, st->syn, st->n_active);
    CK(cudaGetLastError());
    st->has_syn = true;
    return enqueue_syn_pack(st);
}

int qcl_host_alloc(int64_t bytes, void **out) {
    if (!out || bytes < 0) return fail(QCL_EVALUE, "bad argument");
    CK(cudaMallocHost(out, bytes > 0 ? (size_t)bytes : 1));
    return QCL_OK;
}

int qcl_host_free(void *ptr) {
    if (ptr) CK(cudaFreeHost(ptr));
    return QCL_OK;
}

int qcl_state_results(qcl_state *st, uint8_t *words, uint8_t *converged, int64_t *iterations) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    const qcl_plan *p = st->plan;
    DEVICE_SCOPE(p->device);
    if (words && !host_is_pinned(words))  // pageable: pipelined through the pinned ring
        CK(download_bytes(st->ring, words, st->words, (int64_t)st->B * p->n, st->stream));
    else if (words)
        CK(cudaMemcpyAsync(words, st->words, (size_t)st->B * p->n, cudaMemcpyDeviceToHost, st->stream));
    if (converged) CK(cudaMemcpyAsync(converged, st->conv, st->B, cudaMemcpyDeviceToHost, st->stream));
    if (iterations)
        CK(cudaMemcpyAsync(iterations, st->iters, st->B * sizeof(int64_t), cudaMemcpyDeviceToHost, st->stream));
    CK(cudaStreamSynchronize(st->stream));
    return QCL_OK;
}

int qcl_state_info(qcl_state *st, int32_t *lanes, int32_t *flow_engine) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    DEVICE_SCOPE(st->plan->device);
    if (lanes) *lanes = st->W;
    if (flow_engine) {
        // the static conditions first; then the tiling, whose shared-memory fit decides the rest
        bool ok = st->engine == 4 && st->prec == QCL_PREC_FP32 && st->plan->flow_ok && st->plan->max_degree <= 12 &&
                  st->W >= 4;
        if (ok) {
            int rc = ensure_flow(st, 1);
            if (rc) return rc;
            ok = use_flow(st);
        }
        *flow_engine = ok ? 1 : 0;
    }
    return QCL_OK;
}

int qcl_state_kernel_stats(qcl_state *st, int64_t *layer_launches, float *layer_ms, int64_t *all_launches) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    if (layer_launches) *layer_launches = st->launches_layer;
    if (layer_ms) *layer_ms = st->layer_ms;
    if (all_launches) *all_launches = st->launches_all;
    return QCL_OK;
}

int qcl_state_set_engine(qcl_state *st, int32_t engine) {
    if (!st) return fail(QCL_EVALUE, "NULL argument");
    if (st->msg16 && engine != 4 && engine != 6) return msg16_unsupported(st, "engine switch refused");
    if (engine == 4 || engine == 6) {  // flow engine (persistent dataflow decode); 6: with CUDA events
        st->profiling = engine == 6;
        st->engine = 4;
        return QCL_OK;
    }
    if (engine == 2 || engine == 3) {  // engine 0/1 plus CUDA events around every sweep (bench roofline)
        st->profiling = true;
        st->engine = engine - 2;
        if (st->sweep_exec) cudaGraphExecDestroy(st->sweep_exec);
        st->sweep_exec = nullptr;
        return QCL_OK;
    }
    if (engine == 1) {  // direct (register-staged) layer kernels, no TMA pipeline
        st->profiling = false;
        st->engine = 1;
        if (st->sweep_exec) cudaGraphExecDestroy(st->sweep_exec);
        st->sweep_exec = nullptr;
        return QCL_OK;
    }
    if (engine != 0) return fail(QCL_EUNSUP, "engine %d not available", engine);
    st->profiling = false;
    st->engine = engine;
    if (st->sweep_exec) cudaGraphExecDestroy(st->sweep_exec);
    st->sweep_exec = nullptr;
    return QCL_OK;
}

int qcl_decode(qcl_plan *p, const qcl_config *cfg, const void *llr0, int32_t llr_dtype, const uint8_t *syndrome,
               int64_t batch, uint8_t *words, uint8_t *converged, int64_t *iterations) {
    if (!p || !llr0) return fail(QCL_EVALUE, "NULL argument");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    qcl_state *st = nullptr;
    {
        std::lock_guard<std::mutex> lk(p->cache_mu);
        for (size_t i = 0; i < p->cache.size(); i++)
            if (p->cache[i]->B == batch && p->cache[i]->api_prec == cfg->precision) {
                st = p->cache[i];
                p->cache.erase(p->cache.begin() + i);
                break;
            }
    }
    if (!st && (rc = qcl_state_create(p, batch, cfg->precision, &st))) return rc;
    rc = qcl_state_set_llr(st, llr0, llr_dtype);
    if (!rc) rc = qcl_state_set_syndrome(st, syndrome);
    if (!rc) rc = qcl_state_decode(st, cfg, nullptr);
    if (!rc) rc = qcl_state_results(st, words, converged, iterations);
    if (rc) {
        qcl_state_destroy(st);
        return rc;
    }
    std::lock_guard<std::mutex> lk(p->cache_mu);
    if (p->cache.size() < 4)
        p->cache.push_back(st);
    else
        qcl_state_destroy(st);
    return QCL_OK;
}

int qcl_phi(const double *x, int64_t n, double phi_epsilon, double llr_clip, int32_t precision, int32_t device,
            double *out) {
    if (n < 0 || (n > 0 && (!x || !out))) return fail(QCL_EVALUE, "NULL argument");
    if (n == 0) return QCL_OK;
    DEVICE_SCOPE(device);
    double *d = nullptr;
    CK(cudaMalloc(&d, 2 * n * sizeof(double)));
    cudaError_t e = cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        phi_array_kernel<<<(unsigned)cdiv(n, kBlock), kBlock>>>(d, n, phi_epsilon, llr_clip, precision, d + n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d + n, n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(QCL_ECUDA, "qcl_phi: %s", cudaGetErrorString(e));
    return QCL_OK;
}

}  // extern "C"
