"""Host-side mirror of the reference API (no GPU): code model, schedules, channel, sharding,
and the C-ABI library surface (loads, exports every declared symbol, validates plans)."""

import hashlib
import re

import numpy as np
import pytest

import paper_2004_09084_b200 as q
from conftest import (
    CODES,
    GOLDEN,
    MERGE_EXAMPLE_FULL,
    MERGE_EXAMPLE_OUTER_PAIR,
    MERGE_EXAMPLE_TOP_PAIR,
    ROOT,
    TEST_BASE_4x8_Z3,
    random_base_matrix,
)

# ------------------------------------------------------------------ qc_code


@pytest.mark.parametrize(
    "text,match",
    [
        ("", "line 1: malformed header: empty input"),
        ("2 4\n", "line 1: malformed header"),
        ("2 x 3\n", "non-integer field"),
        ("0 4 3\n", "must be positive"),
        ("3 2 4\n0 1\n0 1\n0 1\n", "rows exceed"),
        ("2 3 4\n0 1 2\n", "expected 2 matrix rows"),
        ("1 3 4\n0 1\n", "line 2: expected 3 columns, found 2"),
        ("1 3 4\n0 a 1\n", "non-integer shift"),
        ("1 3 4\n0 4 1\n", "shift out of range"),
        ("1 3 4\n-1 -1 -1\n", "line 2: empty check row"),
    ],
)
def test_parse_errors_match_reference_messages(text, match):
    with pytest.raises(q.MatrixFormatError, match=match):
        q.parse_base_matrix(text)


def test_serialize_roundtrip_and_codes():
    for path in sorted(CODES.glob("*.txt")):
        text = path.read_text()
        base = q.parse_base_matrix(text)
        assert q.serialize_base_matrix(base) == text
    demo = q.load_base_matrix(CODES / "demo_4x8_z100.txt")
    d = q.descriptor(demo)
    assert (d.block_length, d.n_checks, d.rate, d.total_expanded_edges) == (800, 400, 0.5, 2400)


def test_expand_matches_dense_definition():
    rng = np.random.default_rng(3)
    for _ in range(30):
        shifts, z = random_base_matrix(rng)
        base = q.BaseMatrix(len(shifts), len(shifts[0]), z, shifts)
        rows = q.expand(base)
        for i in range(base.n_rows):
            for k in range(z):
                want = sorted(c * z + (k + shifts[i][c]) % z for c in range(base.n_cols) if shifts[i][c] >= 0)
                assert list(rows[i * z + k]) == want


def test_compact_index_order_and_pack():
    base = q.BaseMatrix(3, 3, 4, MERGE_EXAMPLE_OUTER_PAIR)
    sched = q.greedy_schedule(base)
    assert sched.layers == ((0, 2), (1,))
    idx = q.build_compact_index(base, sched)
    assert idx.slot_rows == (0, 2, 1)
    assert idx.slot_offsets == (0, 1, 3, 6)
    assert [(e.shift, e.layer_slot, e.base_col) for e in idx.edges] == [
        (1, 0, 0), (2, 1, 1), (1, 1, 2), (2, 2, 0), (0, 2, 1), (0, 2, 2)]
    shift, col, off, row = idx.packed()
    assert shift.dtype == np.int32 and list(col) == [0, 1, 2, 0, 1, 2] and list(row) == [0, 2, 1]
    with pytest.raises(ValueError, match="partition"):
        q.build_compact_index(base, type("S", (), {"layers": ((0, 1),)})())


def test_greedy_schedule_reference_partitions():
    def sched(shifts):
        return q.greedy_schedule(q.BaseMatrix(3, 3, 4, shifts)).layers

    assert sched(MERGE_EXAMPLE_FULL) == ((0,), (1,), (2,))
    assert sched(MERGE_EXAMPLE_TOP_PAIR) == ((0, 1), (2,))
    assert sched(MERGE_EXAMPLE_OUTER_PAIR) == ((0, 2), (1,))
    with pytest.raises(ValueError):
        q.LayerSchedule(layers=((0,), (0,)))


def test_utilization_and_beta_reference_constants():
    assert abs(q.UtilizationReport(k1=1, k2=128, z=2500).utilization - 0.00477) <= 1e-5
    assert abs(q.beta(0.1, 0.161) - 0.9286) <= 1e-4
    assert abs(q.beta(0.05, 0.076) - 0.9463) <= 1e-4
    assert abs(q.beta(0.02, 0.03) - 0.9380) <= 1e-4


def test_standin_invariants():
    base = q.standin_v2(z=2500)
    assert (base.n_rows, base.n_cols, base.total_edges) == (360, 400, 1507)
    assert q.descriptor(base).total_expanded_edges == 3_767_500
    sched = q.greedy_schedule(base)
    assert [len(l) for l in sched.layers] == [4, 9, 7, 13, 14, 14, 14, 14, 15, 14, 14, 14, 14, 14, 15,
                                              13, 14, 14, 14, 12, 13, 14, 12, 11, 12, 10, 13, 9, 8, 2]
    assert sorted(set((base.shifts >= 0).sum(axis=1).tolist())) == [4, 10, 11]
    assert np.array_equal(q.standin_v2(z=100).shifts >= 0, base.shifts >= 0)
    assert q.serialize_base_matrix(base) == (CODES / "standin_v2_z2500.txt").read_text()


# ------------------------------------------------------------------ channel


def test_channel_mirror_is_bit_exact_with_reference():
    for line in (GOLDEN / "channel_sha.txt").read_text().splitlines():
        seed, snr, snr_idx, frame, n, sha = line.split()
        chan = q.ChannelConfig(snr=float(snr), seed=int(seed))
        llr = q.init_llr(q.transmit(np.zeros(int(n), np.uint8), chan, q.frame_rng(int(seed), int(snr_idx), int(frame))), chan)
        assert hashlib.sha256(llr.tobytes()).hexdigest() == sha
    with pytest.raises(ValueError):
        q.ChannelConfig(snr=0.0)


def test_decoder_config_validation():
    with pytest.raises(ValueError):
        q.DecoderConfig(max_iterations=0)
    with pytest.raises(ValueError):
        q.DecoderConfig(llr_clip=0.0)
    with pytest.raises(ValueError):
        q.DecoderConfig(phi_epsilon=1.5)


def test_syndrome_of_host_utility():
    base = q.BaseMatrix(4, 8, 3, TEST_BASE_4x8_Z3)
    rows = q.expand(base)
    for j in (0, 7, 23):
        w = np.zeros(24, np.uint8)
        w[j] = 1
        assert np.array_equal(q.syndrome_of(w, rows).astype(bool), np.array([j in r for r in rows]))


# ------------------------------------------------------------------ sharding


def test_shard_ranges_follow_array_split():
    from paper_2004_09084_b200.sharding import shard_range

    for total in (1, 7, 64, 513):
        for world in (1, 2, 3, 8):
            parts = np.array_split(np.arange(total), world)
            for r in range(world):
                a, b = shard_range(total, world, r)
                assert (a, b) == ((int(parts[r][0]), int(parts[r][-1]) + 1) if parts[r].size else (a, a))


# ------------------------------------------------------------------ C ABI surface (no GPU)


def test_library_loads_and_exports_every_declared_symbol():
    import ctypes

    from paper_2004_09084_b200 import _native

    lib = _native.lib()
    header = (ROOT / "include" / "qcldpc_b200.h").read_text()
    declared = set(re.findall(r"\b(qcl_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_native.EXPORTED) == declared
    assert lib.qcl_abi_version() == 1
    # the library is the in-tree build (what the driver records as loaded)
    assert _native.LIB_PATH.parent == ROOT / "paper_2004_09084_b200"
    assert isinstance(lib, ctypes.CDLL)


def test_plan_validation_messages_without_gpu():
    """Validation runs before any CUDA call, with the reference's ValueError texts."""
    from paper_2004_09084_b200 import _native

    base = q.BaseMatrix(3, 3, 4, MERGE_EXAMPLE_OUTER_PAIR)
    index = q.build_compact_index(base, q.single_row_schedule(base))
    with pytest.raises(ValueError, match="does not match"):
        q.LayeredDecoder(index, q.greedy_schedule(base), q.DecoderConfig())
    # merged rows sharing a column: construct a bad schedule/index pair by hand
    bad_base = q.BaseMatrix(2, 2, 3, [[0, 1], [1, -1]])
    bad_sched = type("Sched", (), {"layers": ((0, 1),)})()
    bad_index = q.build_compact_index(bad_base, q.LayerSchedule(layers=((0, 1),)))
    with pytest.raises(ValueError, match="rows within a layer share a base column"):
        _native.Plan(bad_index, bad_sched, 0)


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle or computes decodes in numpy."""
    pkg = ROOT / "paper_2004_09084_b200"
    for path in pkg.glob("*.py"):
        text = path.read_text()
        assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", text), path.name
