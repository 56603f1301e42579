"""The flow engine (engine 4: one persistent launch per decode, tiles ordered by
per-tile completion flags, csrc/flow.cuh) against the per-layer engine (0).

Both engines run the same FP32 check-node arithmetic on the same tiles, so with the
layer order preserved by the flags the results must be BIT-IDENTICAL: any missing
dependency edge or memory-ordering hole shows up as a mismatch.  Decodes are repeated
(the schedule is dynamic, so every run interleaves tiles differently) and start from
fresh states (the upload path that once raced with the first launch).
"""

import numpy as np
import pytest

from conftest import ROOT, channel_llrs, load_code

pytestmark = pytest.mark.gpu


def _states(name, batch, seed=3, syndrome=False):
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code(name)
    plan = _native.Plan(index, sched, 0)
    out = []
    m = base.n_rows * base.z
    syn = None
    if syndrome:
        syn = (np.random.default_rng(seed).random((batch, m)) < 0.5).astype(np.uint8)
    for engine in (0, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=seed, snr_idx=0, first_frame=0, snr=0.161)
        st.set_syndrome(syn)
        out.append(st)
    return base, sched, out


@pytest.mark.parametrize("name,batch,iters", [("standin_v2_z100", 64, 20), ("standin_v2_z2500", 64, 4),
                                              ("standin_v2_z100", 8, 30), ("demo_6x12_z16", 33, 12),
                                              ("standin_v2_z100", 256, 12), ("standin_v2_z2500", 128, 3),
                                              ("standin_v2_z100", 192, 6), ("standin_v2_z100", 200, 6)])
def test_flow_decode_bit_identical_to_layer_engine(gpu, name, batch, iters):
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    _, _, (ref, flow) = _states(name, batch)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=iters, early_termination=False), "fp32")
    ref.decode(cfg)
    want = ref.download()
    want_res = ref.results()
    for trial in range(4):  # dynamic tile schedule: every run interleaves differently
        flow.decode(cfg)
        got = flow.download()
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), trial
        for a, b in zip(flow.results(), want_res):
            assert np.array_equal(a, b), trial


def test_flow_sweeps_with_syndrome(gpu):
    """Whole sweeps through qcl_state_layers (the flow path of _sweep) with a random target."""
    _, sched, (ref, flow) = _states("standin_v2_z100", 16, syndrome=True)
    for st in (ref, flow):
        st.reset(30.0)
        for _ in range(5):
            st.layers(0, len(sched.layers), 30.0, 1e-10)
    a, b = ref.download(), flow.download()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("snr", [0.161, 0.2])
def test_flow_early_termination_matches(gpu, snr):
    """ET decodes (one flow launch per sweep): words, flags and iteration counts identical."""
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, snr, 0, 0, 48)
    cfg = q.DecoderConfig(max_iterations=50, early_termination=True)
    res = [q.LayeredDecoder(index, sched, cfg, engine=e).decode_batch_arrays(llr, np.zeros((48, m), np.uint8))
           for e in (0, 4)]
    for a, b in zip(*res):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("batch,snr", [(64, 0.18), (128, 0.2), (21, 0.19)])
def test_fused_early_termination_repeated(gpu, batch, snr):
    """ET inside the flow launch (flow.cuh, "Fused early termination"): random codewords
    with their nonzero targets (encode mode), one and two group blocks, a ragged lane group; repeated decodes (every run
    interleaves tiles, checks and decisions differently) equal the per-layer engine's
    per-sweep check: words, converged flags, iteration counts."""
    from paper_2004_09084_b200 import _native
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=40, early_termination=True), "fp32")
    outs = []
    for engine in (0, 4, 4, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=5, snr_idx=1, first_frame=0, snr=snr, encode_mode=True)  # random words, H c
        st.decode(cfg)
        outs.append(st.results())
    want = outs[0]
    assert want[1].any()  # some frames converge, some (possibly) do not
    for got in outs[1:]:
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_flow_fresh_states_first_launch(gpu):
    """A new decoder's first decode (table uploads immediately followed by the launch)."""
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 0.161, 0, 0, 64)
    cfg = q.DecoderConfig(max_iterations=12, early_termination=False)
    want = q.LayeredDecoder(index, sched, cfg, engine=0).decode_batch_arrays(llr, np.zeros((64, m), np.uint8))
    for _ in range(3):
        got = q.LayeredDecoder(index, sched, cfg, engine=4).decode_batch_arrays(llr, np.zeros((64, m), np.uint8))
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def _high_degree_code():
    """3 x 20 base matrix with row degrees 16 / 14 / 20 (above the flow engine's 12), z = 24."""
    from conftest import make_code

    rng = np.random.default_rng(11)
    shifts = np.full((3, 20), -1, dtype=np.int64)
    for i, deg in enumerate((16, 14, 20)):
        cols = rng.choice(20, size=deg, replace=False)
        shifts[i, cols] = rng.integers(0, 24, size=deg)
    return make_code(shifts.tolist(), 24, merged=True)


def test_high_degree_codes_fall_back_to_the_layer_engine(gpu):
    """Row degree > 12: the default engine runs the per-layer kernels, with results equal
    to engine 0 and to the FP64 path's decisions on a clean channel; FP16 messages refuse."""
    import paper_2004_09084_b200 as q

    base, sched, index = _high_degree_code()
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 4.0, seed=2, snr_idx=0, frames=16)
    syn = np.zeros((16, m), np.uint8)
    cfg = q.DecoderConfig(max_iterations=8, early_termination=True)
    out = {e: q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=e).decode_batch_arrays(llr, syn)
           for e in (0, 4)}
    for a, b in zip(out[0], out[4]):
        assert np.array_equal(a, b)
    ref = q.LayeredDecoder(index, sched, cfg, precision="fp64").decode_batch_arrays(llr, syn)
    assert np.array_equal(ref[1], out[4][1]) and np.array_equal(ref[2], out[4][2])
    with pytest.raises(RuntimeError, match="flow engine"):
        q.LayeredDecoder(index, sched, cfg, precision="fp32-msg16").decode_batch_arrays(llr, syn)


def test_random_codes_all_engines_agree(gpu):
    """40 random codes (row degrees 1..20, z 1..40, merged or single-row schedules), random
    targets, 8..136 codewords (1..17 lane groups, two group blocks at 128): the flow engine,
    the TMA and the direct per-layer engines give bit-identical decodes (ET on and off) and
    states; FP16 messages run wherever the flow engine does, and refuse cleanly elsewhere."""
    import paper_2004_09084_b200 as q
    from conftest import make_code

    rng = np.random.default_rng(7)
    for trial in range(40):
        n_rows = int(rng.integers(1, 6))
        n_cols = int(rng.integers(n_rows + 1, 24))
        z = int(rng.integers(1, 41))
        shifts = np.full((n_rows, n_cols), -1, dtype=np.int64)
        for i in range(n_rows):
            deg = int(rng.integers(1, min(20, n_cols) + 1))
            cols = rng.choice(n_cols, size=deg, replace=False)
            shifts[i, cols] = rng.integers(0, z, size=deg)
        base, sched, index = make_code(shifts.tolist(), z, merged=bool(trial % 2))
        batch = (8, 24, 72, 128, 136)[trial % 5]
        n, m = base.n_cols * z, base.n_rows * z
        llr = rng.normal(0.8, 2.0, size=(batch, n))
        syn = (rng.random((batch, m)) < 0.2).astype(np.uint8)
        cfg = q.DecoderConfig(max_iterations=6, early_termination=bool(trial % 3))
        outs = [q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=e).decode_batch_arrays(llr, syn)
                for e in (0, 1, 4)]
        for o in outs[1:]:
            for a, b in zip(outs[0], o):
                assert np.array_equal(a, b), trial
        flow_ok = max(len([s for s in row if s >= 0]) for row in shifts.tolist()) <= 12
        if flow_ok:
            w, c, it = q.LayeredDecoder(index, sched, cfg, precision="fp32-msg16").decode_batch_arrays(llr, syn)
            assert w.shape == outs[0][0].shape and np.all(it >= 1), trial
        else:
            with pytest.raises(RuntimeError, match="flow engine"):
                q.LayeredDecoder(index, sched, cfg, precision="fp32-msg16").decode_batch_arrays(llr, syn)


def test_one_decoder_shared_by_threads(gpu):
    """decoder.py:18-21 / :469-472: one decoder instance used by several host threads at
    once (each call gets its own state, stream, flags and claim counters): results equal
    the sequential calls', for FP32 and FP16 messages."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    batches = [channel_llrs(n, 0.2, seed=3, snr_idx=0, frames=16, start=16 * i) for i in range(8)]
    syn = np.zeros((16, m), np.uint8)
    for precision in ("fp32", "fp32-msg16"):
        for et in (True, False):
            dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=15, early_termination=et),
                                   precision=precision)
            want = [dec.decode_batch_arrays(b, syn) for b in batches]
            with ThreadPoolExecutor(4) as ex:
                got = list(ex.map(lambda b: dec.decode_batch_arrays(b, syn), batches))
            for w, g in zip(want, got):
                for a, b in zip(w, g):
                    assert np.array_equal(a, b), (precision, et)


@pytest.mark.parametrize("z", [37, 40, 101, 128])
def test_fused_et_converging_frames_nonzero_targets(gpu, z):
    """Fused early termination where frames converge at different sweeps toward nonzero
    targets (s = H x for a random word x, LLRs pointing at x with noise): the check items'
    word-wise scan (z % 4 == 0) and byte scan (z odd), the last-failed-check hints and the
    shared early exit all feed the decisions; outcomes equal the per-layer engine's bit for
    bit and every converged word satisfies its target."""
    import paper_2004_09084_b200 as q
    from conftest import make_code

    rng = np.random.default_rng(z)
    n_rows, n_cols = 6, 16
    shifts = np.full((n_rows, n_cols), -1, dtype=np.int64)
    for i in range(n_rows):
        cols = rng.choice(n_cols, size=int(rng.integers(3, 9)), replace=False)
        shifts[i, cols] = rng.integers(0, z, size=len(cols))
    base, sched, index = make_code(shifts.tolist(), z, merged=True)
    n, m = n_cols * z, n_rows * z
    B = 72
    x = (rng.random((B, n)) < 0.5).astype(np.uint8)
    rows = q.expand(base)
    syn = np.stack([x[:, r].sum(axis=1) & 1 for r in rows], axis=1).astype(np.uint8)
    # per-frame noise level: some frames converge in a sweep or two, others late or never
    sigma = rng.uniform(0.5, 1.1, size=(B, 1))
    llr = (1.0 - 2.0 * x) * 2.0 / sigma**2 + rng.normal(0.0, 1.0, size=(B, n)) * 2.0 / sigma
    cfg = q.DecoderConfig(max_iterations=30, early_termination=True)
    want = q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=0).decode_batch_arrays(llr, syn)
    got = q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=4).decode_batch_arrays(llr, syn)
    for a, b in zip(want, got):
        assert np.array_equal(a, b)
    w, c, it = got
    print(f"z={z}: {int(c.sum())}/{B} converged, iterations {np.bincount(it).nonzero()[0].tolist()}")
    assert 5 < c.sum() < B - 5 and len(set(it[c].tolist())) >= 3  # a spread of convergence sweeps
    got_syn = np.stack([w[:, r].sum(axis=1) & 1 for r in rows], axis=1).astype(np.uint8)
    assert np.array_equal(got_syn[c], syn[c])


@pytest.mark.parametrize("batch,snr", [(128, 1.5), (21, 1.5), (64, 1.0), (136, 1.0), (40, 1.2)])
def test_fused_et_all_frames_converge(gpu, batch, snr):
    """Fused ET where every frame converges well before the cap: the static-order kernel's
    CTAs stop taking items and every wait that points at a stopped CTA's tile is abandoned
    (flow.cuh kSpinAborted / consumers_sync_or).  Repeated decodes must terminate and equal
    the per-layer engine's per-sweep check bit for bit."""
    from paper_2004_09084_b200 import _native
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=True), "fp32")
    outs = []
    for engine in (0, 4, 4, 4, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=9, snr_idx=2, first_frame=0, snr=snr, encode_mode=True)
        st.decode(cfg)
        outs.append(st.results())
    want = outs[0]
    assert want[1].all() and want[2].max() < 50, (want[1].mean(), want[2].max())  # every frame converged early
    for got in outs[1:]:
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
