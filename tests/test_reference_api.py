"""The reference's behavioural decoder tests (pkg/tests/test_decoder.py), run against the
CUDA drop-in through its public API.  Each test names the reference test it mirrors.
Independent checks (dense expansion, tanh-product check node, exhaustive ML) are
re-implemented here, sharing no code with the package."""

import math

import numpy as np
import pytest

import paper_2004_09084_b200 as q
from conftest import MERGE_EXAMPLE_OUTER_PAIR, MERGE_EXAMPLE_TOP_PAIR, TEST_BASE_4x8_Z3, make_code

pytestmark = pytest.mark.gpu
PRECISIONS = ["fp64", "fp32"]
TOL = {"fp64": 1e-9, "fp32": 2e-5}


def dense_h(shifts, z):
    s = np.asarray(shifts)
    h = np.zeros((s.shape[0] * z, s.shape[1] * z), np.uint8)
    for i in range(s.shape[0]):
        for c in range(s.shape[1]):
            if s[i, c] >= 0:
                for k in range(z):
                    h[i * z + k, c * z + (k + s[i, c]) % z] = 1
    return h


def tanh_check(incoming, bit):
    x = np.asarray(incoming, dtype=np.float64)
    out = np.array([2 * np.arctanh(np.clip(np.prod(np.tanh(np.delete(x, j) / 2)), -1 + 1e-15, 1 - 1e-15))
                    for j in range(len(x))])
    return -out if bit else out


def ml_decode(h, s, llr):
    """Exhaustive syndrome-constrained ML over GF(2) (tiny codes only)."""
    m, n = h.shape
    a = np.concatenate([h % 2, np.asarray(s, np.uint8)[:, None] % 2], axis=1).astype(np.uint8)
    piv, r = [], 0
    for c in range(n):
        hit = [i for i in range(r, m) if a[i, c]]
        if not hit:
            continue
        a[[r, hit[0]]] = a[[hit[0], r]]
        for i in range(m):
            if i != r and a[i, c]:
                a[i] ^= a[r]
        piv.append(c)
        r += 1
    x0 = np.zeros(n, np.uint8)
    for i, c in enumerate(piv):
        x0[c] = a[i, n]
    free = [c for c in range(n) if c not in piv]
    basis = []
    for f in free:
        v = np.zeros(n, np.uint8)
        v[f] = 1
        for i, c in enumerate(piv):
            v[c] = a[i, f]
        basis.append(v)
    best, best_m = None, -np.inf
    for mask in range(1 << len(basis)):
        x = x0.copy()
        for j, v in enumerate(basis):
            if mask >> j & 1:
                x ^= v
        metric = float(np.sum((1.0 - 2.0 * x) * llr))
        if metric > best_m:
            best, best_m = x, metric
    return best


def channel(base, snr, seed):
    n = base.n_cols * base.z
    cfg = q.ChannelConfig(snr=snr, seed=seed)
    return q.init_llr(q.transmit(np.zeros(n, np.uint8), cfg), cfg)


# ------------------------------------------------------------------ phi (test_decoder.py:58-82)


def test_phi_reference_values(gpu):
    assert q.phi(2.0) == pytest.approx(-math.log(math.tanh(1.0)), rel=1e-12)
    x = np.logspace(np.log10(0.1), np.log10(20.0), 10_000)
    assert np.max(np.abs(q.phi(q.phi(x)) - x) / x) < 1e-9
    xs = np.linspace(0.3, 8.0, 57)
    assert np.allclose(q.phi(xs), -np.log(np.tanh(xs / 2.0)), rtol=1e-12)
    assert q.phi(0.0) == q.phi(1e-10) and q.phi(1e6) == q.phi(30.0)
    assert np.allclose(q.phi(xs, precision="fp32"), -np.log(np.tanh(xs / 2.0)), rtol=3e-6)


# ------------------------------------------------------------------ layer update


@pytest.mark.parametrize("precision", PRECISIONS)
def test_degree_two_check_is_passthrough(gpu, precision):  # test_decoder.py:97-110
    base, sched, index = make_code([[0, 0]], z=1)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(), precision=precision)
    a, b = 1.2, 0.8
    st = dec.new_state(np.array([a, b]))
    dec.layer_update(st, 0, np.array([0]))
    assert st.edge_messages[0] == pytest.approx([b, a], rel=TOL[precision])
    assert st.posterior[0] == pytest.approx([a + b, a + b], rel=TOL[precision])
    st = dec.new_state(np.array([a, b]))
    dec.layer_update(st, 0, np.array([1]))
    assert st.edge_messages[0] == pytest.approx([-b, -a], rel=TOL[precision])


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("bit", [0, 1])
@pytest.mark.parametrize("inputs", [(1.5, 0.9, 2.4), (-1.1, 0.6, 3.0), (0.4, -0.4, -2.2), (5.0, 4.0, 3.0)])
def test_single_check_matches_tanh_product(gpu, inputs, bit, precision):  # :113-124
    base, sched, index = make_code([[0, 0, 0]], z=1)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(), precision=precision)
    st = dec.new_state(np.array(inputs))
    dec.layer_update(st, 0, np.array([bit]))
    assert np.allclose(st.edge_messages[0], tanh_check(inputs, bit), rtol=TOL[precision], atol=1e-6)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_ragged_merged_layer_and_degree_one_check(gpu, precision):  # :127-144
    base, sched, index = make_code([[0, 0, -1], [-1, -1, 0]], z=1, merged=True)
    assert sched.layers == ((0, 1),)
    cfg = q.DecoderConfig()
    dec = q.LayeredDecoder(index, sched, cfg, precision=precision)
    pinned = q.phi(cfg.phi_epsilon)
    for syn in ([0, 0], [1, 0], [0, 1], [1, 1]):
        st = dec.new_state(np.array([1.1, -0.4, 0.7]))
        dec.layer_update(st, 0, np.array(syn, dtype=np.uint8))
        assert st.edge_messages[0, :2] == pytest.approx(tanh_check([1.1, -0.4], syn[0]), rel=TOL[precision])
        sign = -1.0 if syn[1] else 1.0
        assert st.edge_messages[0, 2] == pytest.approx(sign * pinned, rel=TOL[precision])


def test_layer_update_only_touches_layer_variables(gpu):  # :147-165
    base, sched, index = make_code(MERGE_EXAMPLE_TOP_PAIR, z=5, merged=True)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig())
    llr = q.frame_rng(0).normal(size=15)
    st = dec.new_state(llr)
    before = st.posterior.copy()
    dec.layer_update(st, 0, np.zeros(15, np.uint8))
    assert not np.array_equal(st.posterior, before)
    lo, hi = dec._slot_edge_span[2]
    assert not st.edge_messages[0, lo:hi].any()


@pytest.mark.parametrize("precision", PRECISIONS)
def test_state_invariants_after_updates(gpu, precision):  # :168-181
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    cfg = q.DecoderConfig(llr_clip=8.0)
    dec = q.LayeredDecoder(index, sched, cfg, precision=precision)
    st = dec.new_state(np.array([1e308, -1e308, 0.0, 1e-300, -5.0, 42.0] * 4))
    syn = q.frame_rng(1).integers(0, 2, size=12).astype(np.uint8)
    for _ in range(3):
        for layer in range(len(sched.layers)):
            dec.layer_update(st, layer, syn)
            assert np.isfinite(st.posterior).all() and np.abs(st.posterior).max() <= 8.0
            assert np.isfinite(st.edge_messages).all() and np.abs(st.edge_messages).max() <= 8.0


# ------------------------------------------------------------------ decoding


@pytest.mark.parametrize("precision", PRECISIONS)
def test_noiseless_zero_word_converges_immediately(gpu, precision):  # :209-220
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    out = q.decode(np.full(24, 20.0), np.zeros(12, np.uint8), index, sched, q.DecoderConfig(max_iterations=10),
                   precision=precision)
    assert out.converged and out.iterations_used == 1 and not out.word.any()


@pytest.mark.parametrize("precision", PRECISIONS)
def test_single_flip_corrected_and_matches_ml(gpu, precision):  # :230-242
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    h = dense_h(base.shifts, base.z)
    rng = q.frame_rng(99)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(), precision=precision)
    for _ in range(20):
        flip = int(rng.integers(0, 24))
        llr = np.full(24, 7.0)
        llr[flip] = -4.0
        w, c, it = dec.decode_batch_arrays(llr[None], np.zeros((1, 12), np.uint8))
        assert c[0] and not w.any()
        assert np.array_equal(w[0], ml_decode(h, np.zeros(12, np.uint8), llr))


@pytest.mark.parametrize("precision", PRECISIONS)
def test_decode_toward_nonzero_syndrome(gpu, precision):  # :245-255, :323-335
    for shifts, z, merged, n in [(TEST_BASE_4x8_Z3, 3, False, 24), (MERGE_EXAMPLE_TOP_PAIR, 5, True, 15)]:
        base, sched, index = make_code(shifts, z, merged=merged)
        rows = q.expand(base)
        word = q.frame_rng(3).integers(0, 2, size=n).astype(np.uint8)
        syn = q.syndrome_of(word, rows)
        out = q.decode(9.0 * (1.0 - 2.0 * word), syn, index, sched, q.DecoderConfig(), precision=precision)
        assert out.converged and np.array_equal(out.word, word)


def test_converged_implies_syndrome_satisfied(gpu):  # :258-265
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    rows = q.expand(base)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=20))
    for seed in range(60):
        w, c, _ = dec.decode_batch_arrays(channel(base, 1.5, seed)[None], np.zeros((1, 12), np.uint8))
        if c[0]:
            assert not q.syndrome_of(w[0], rows).any()


@pytest.mark.parametrize("precision", PRECISIONS)
def test_syndrome_sign_symmetry_is_bit_exact(gpu, precision):  # :268-282
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    rows = q.expand(base)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=25), precision=precision)
    rng = q.frame_rng(17)
    for seed in range(25):
        llr = channel(base, 1.2, 1000 + seed)
        e = (rng.random(24) < 0.2).astype(np.uint8)
        w0, c0, i0 = dec.decode_batch_arrays(llr[None], np.zeros((1, 12), np.uint8))
        w1, c1, i1 = dec.decode_batch_arrays((llr * (1.0 - 2.0 * e))[None], q.syndrome_of(e, rows)[None])
        assert np.array_equal(w1[0], w0[0] ^ e) and i1[0] == i0[0] and c1[0] == c0[0]


def test_early_termination_stability_one_extra_iteration(gpu):  # :285-304
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    rows = q.expand(base)
    tested = 0
    for seed in range(40):
        llr = channel(base, 1.8, seed)
        out = q.decode(llr, np.zeros(12, np.uint8), index, sched, q.DecoderConfig(max_iterations=30))
        if not out.converged:
            continue
        longer = q.decode(llr, np.zeros(12, np.uint8), index, sched,
                          q.DecoderConfig(max_iterations=out.iterations_used + 1, early_termination=False))
        assert longer.converged and not q.syndrome_of(longer.word, rows).any()
        tested += 1
    assert tested > 10


def test_decode_validates_shapes(gpu):  # :307-312
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    with pytest.raises(ValueError, match="block length"):
        q.decode(np.zeros(23), np.zeros(12, np.uint8), index, sched, q.DecoderConfig())
    with pytest.raises(ValueError, match="syndrome shape"):
        q.decode(np.zeros(24), np.zeros(11, np.uint8), index, sched, q.DecoderConfig())


def test_decoder_rejects_mismatched_schedule(gpu):  # :315-320
    base = q.BaseMatrix(3, 3, 4, MERGE_EXAMPLE_OUTER_PAIR)
    index = q.build_compact_index(base, q.single_row_schedule(base))
    with pytest.raises(ValueError, match="does not match"):
        q.LayeredDecoder(index, q.greedy_schedule(base), q.DecoderConfig())


# ------------------------------------------------------------------ batching (:341-386)


def test_batch_is_bit_identical_to_sequential_and_worker_invariant(gpu):
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    cfg = q.DecoderConfig(max_iterations=15)
    frames = [(channel(base, 1.5, s), np.zeros(12, np.uint8)) for s in range(32)]
    batch = q.decode_batch(frames, index, sched, cfg)
    for frame, out in zip(frames, batch):
        single = q.decode(frame[0], frame[1], index, sched, cfg)
        assert np.array_equal(single.word, out.word)
        assert (single.converged, single.iterations_used) == (out.converged, out.iterations_used)
    perm = q.frame_rng(2).permutation(len(frames))
    permuted = q.decode_batch([frames[i] for i in perm], index, sched, cfg)
    for where, i in enumerate(perm):
        assert np.array_equal(permuted[where].word, batch[i].word)
    for workers in (2, 4):
        threaded = q.decode_batch(frames, index, sched, cfg, workers=workers)
        for a, b in zip(batch, threaded):
            assert np.array_equal(a.word, b.word) and a.iterations_used == b.iterations_used
    assert q.decode_batch([], index, sched, cfg) == []


def test_reference_objects_are_accepted_duck_typed(gpu):
    """The decoder takes any CompactIndex/LayerSchedule-shaped objects (decoder.py:117-189)."""
    base, sched, index = make_code(TEST_BASE_4x8_Z3, z=3)
    Sched = type("Sched", (), {"layers": sched.layers})
    dec = q.LayeredDecoder(index, Sched(), q.DecoderConfig(max_iterations=5))
    w, c, it = dec.decode_batch_arrays(np.full((2, 24), 9.0), np.zeros((2, 12), np.uint8))
    assert c.all() and (it == 1).all() and not w.any()
