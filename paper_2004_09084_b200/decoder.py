"""Layered BP decoding toward a target syndrome, on B200 (drop-in for ``qcldpc.decoder``).

Same public surface as ``/root/reference/pkg/src/qcldpc/decoder.py`` -- DecoderConfig,
DecodeOutcome, DecoderState, phi, LayeredDecoder{new_state, layer_update,
hard_decision, syndrome_satisfied, decode_batch_arrays}, decode, decode_batch --
with the same argument meaning, shapes, dtypes and ValueError texts.  Every
numeric operation runs in ``libqcldpc_b200.so`` (hand-written sm_100a CUDA behind a
C ABI); this module only validates arguments, moves arrays across the ABI and
shapes results.

Three precisions, chosen per decoder:
  * ``precision="fp32"`` (default) -- the performance path: FP32 posteriors and edge
    messages, exclusive Phi-sums, fast Phi (``csrc/phi.cuh``).
  * ``precision="fp64"`` -- the parity path: FP64 state, the reference's own
    ``total - own`` formula and numpy fold order, libdevice log1p/expm1.
  * ``precision="fp32-msg16"`` -- opt-in, beyond parity: FP32 posteriors, FP16 edge
    messages (12 instead of 16 bytes per edge and iteration).  Whole decodes and whole
    sweeps on the flow engine only; its decisions are not bit-identical to ``"fp32"``
    (FER parity is statistical).

Extra keywords beyond the reference: ``device`` (CUDA ordinal) and ``precision``.
``ShardedDecoder`` spreads a batch over several GPUs of one process
(contiguous slices, no collective), the device analogue of
``decode_batch(..., workers)`` (``decoder.py:453-476``).
"""

from __future__ import annotations

import threading
from collections import deque
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "DecodeOutcome",
    "DecoderConfig",
    "DecoderState",
    "LayeredDecoder",
    "ShardedDecoder",
    "decode",
    "decode_batch",
    "phi",
    "syndrome_of",
]

DEFAULT_LLR_CLIP = 30.0
DEFAULT_PHI_EPSILON = 1e-10


@dataclass(frozen=True)
class DecoderConfig:
    """Iteration budget, termination policy, numeric guards (``decoder.py:48-63``)."""

    max_iterations: int = 50
    early_termination: bool = True
    llr_clip: float = DEFAULT_LLR_CLIP
    phi_epsilon: float = DEFAULT_PHI_EPSILON

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if not self.llr_clip > 0:
            raise ValueError("llr_clip must be positive")
        if not 0 < self.phi_epsilon < 1:
            raise ValueError("phi_epsilon must be in (0, 1)")


@dataclass
class DecodeOutcome:
    """Hard decision, whether it meets the target syndrome, iterations used."""

    word: np.ndarray
    converged: bool
    iterations_used: int


@dataclass
class DecoderState:
    """Host view of a decoding state in the reference layout (``decoder.py:75-93``).

    ``posterior`` is (batch, n) float64; ``edge_messages`` is (batch, total_edges*z)
    float64, slot by slot, each slot an (edge, z-offset) block.
    """

    posterior: np.ndarray
    edge_messages: np.ndarray
    iteration: int = 0
    layer: int = -1

    @property
    def batch_size(self):
        return self.posterior.shape[0]


def phi(x, phi_epsilon=DEFAULT_PHI_EPSILON, llr_clip=DEFAULT_LLR_CLIP, precision="fp64", device=0):
    """-ln tanh(x/2) as the device kernels evaluate it (``decoder.py:96-105``).

    ``precision="fp64"`` is the parity path's libdevice log1p(2/expm1(x));
    ``"fp32"`` is the performance path's three-region MUFU evaluation.
    """
    out = _native.phi_device(x, phi_epsilon, llr_clip, precision, device)
    return out if np.ndim(x) else float(out)


def _as_cfg(cfg):
    # accept the reference's DecoderConfig (duck-typed) as well as ours
    return DecoderConfig(
        max_iterations=int(cfg.max_iterations),
        early_termination=bool(cfg.early_termination),
        llr_clip=float(cfg.llr_clip),
        phi_epsilon=float(cfg.phi_epsilon),
    )


class LayeredDecoder:
    """Compiled layered decoder for one (compact index, schedule) pair on one GPU.

    Construction mirrors ``decoder.py:117-189``: the schedule must match the index
    row order and rows merged into a layer must touch disjoint base columns (both
    checked again by ``qcl_plan_create``).  The packed ``H_compact1`` table is uploaded
    once; device workspaces are cached per host thread and batch size, so one
    instance can be shared by a ThreadPoolExecutor like the reference's.
    """

    def __init__(self, index, schedule, cfg, device=0, precision="fp32", engine=4):
        flat_rows = tuple(r for layer in schedule.layers for r in layer)
        if flat_rows != tuple(index.slot_rows):
            raise ValueError("schedule does not match the compact index row order")
        if precision not in _native.PREC:
            raise ValueError(f"precision must be one of {sorted(_native.PREC)}")
        self.cfg = _as_cfg(cfg)
        self.index = index
        self.schedule = schedule
        self.precision = precision
        self.engine = int(engine)  # 4: flow engine (default), 0: TMA per-layer kernels, 1: direct kernels
        self.device = int(device)
        self.z = int(index.z)
        self.n_vars = int(index.n_cols) * self.z
        self.n_checks = len(index.slot_rows) * self.z
        z = self.z
        self._slot_edge_span = [
            (index.slot_offsets[s] * z, index.slot_offsets[s + 1] * z) for s in range(len(index.slot_rows))
        ]
        # layer-safety check + device upload (ValueError texts from decoder.py:120,152)
        self._plan = _native.Plan(index, schedule, self.device)
        self._qcfg = _native.make_config(self.cfg, precision)
        self._local = threading.local()

    # ------------------------------------------------------------------ workspaces
    def _state(self, batch):
        cache = getattr(self._local, "states", None)
        if cache is None:
            cache = self._local.states = {}
        st = cache.get(batch)
        if st is None:
            if len(cache) >= 4:
                cache.clear()
            st = cache[batch] = _native.State(self._plan, batch, self.precision)
            st.set_engine(self.engine)
        return st

    # ------------------------------------------------------------------ state API
    def new_state(self, llr0):
        """posterior = clip(llr0), messages = 0 (``decoder.py:191-202``)."""
        posterior = np.atleast_2d(np.asarray(llr0, dtype=np.float64)).copy()
        if posterior.shape[1] != self.n_vars:
            raise ValueError(f"llr vector length {posterior.shape[1]} != block length {self.n_vars}")
        st = self._state(posterior.shape[0])
        st.set_llr(posterior)
        st.reset(self.cfg.llr_clip)
        post, msg = st.download()
        return DecoderState(posterior=post, edge_messages=msg)

    def _check_syndrome(self, syndrome, batch):
        syndrome = np.atleast_2d(np.asarray(syndrome))
        if syndrome.shape != (batch, self.n_checks):
            raise ValueError(f"syndrome shape {syndrome.shape} != ({batch}, {self.n_checks})")
        return syndrome.astype(bool)

    def _run_layers(self, state, first, count, syndrome):
        syn = self._check_syndrome(syndrome, state.batch_size)
        st = self._state(state.batch_size)
        st.upload(state.posterior, state.edge_messages)
        st.set_syndrome(syn.view(np.uint8))
        st.layers(first, count, self.cfg.llr_clip, self.cfg.phi_epsilon)
        post, msg = st.download()
        state.posterior[...] = post
        state.edge_messages[...] = msg

    def layer_update(self, state, layer, syndrome):
        """Apply one layer's check updates to the state, in place (``decoder.py:252-257``)."""
        if not 0 <= int(layer) < len(self.schedule.layers):
            raise IndexError(f"layer {layer} out of range")
        self._run_layers(state, int(layer), 1, syndrome)
        state.layer = int(layer)
        return state

    def _sweep(self, state, syndrome):
        self._run_layers(state, 0, len(self.schedule.layers), syndrome)
        state.layer = len(self.schedule.layers) - 1

    def hard_decision(self, state):
        """Bit 0 wherever the posterior is >= 0 (``decoder.py:264-266``)."""
        st = self._state(state.batch_size)
        st.upload(state.posterior, None)
        return st.hard_decision()

    def syndrome_satisfied(self, words, syndrome):
        """Per-frame H @ word == syndrome over GF(2) (``decoder.py:268-273``)."""
        words = np.atleast_2d(np.asarray(words))
        syn = self._check_syndrome(syndrome, words.shape[0])
        st = self._state(words.shape[0])
        # posterior = +-1 carries exactly the word's bits into the device check
        st.upload(np.where(words.astype(bool), -1.0, 1.0), None)
        st.set_syndrome(syn.view(np.uint8))
        return st.syndrome_ok()

    # ------------------------------------------------------------------ decode
    def decode_batch_arrays(self, llr0, syndrome):
        """Decode a (batch, n) LLR block toward (batch, m) syndromes (``decoder.py:275-312``).

        float32 LLRs are passed through as-is (half the host->device bytes); anything
        else is coerced to float64 like the reference.
        """
        llr = np.atleast_2d(np.asarray(llr0))
        if llr.dtype != np.float32:
            llr = llr.astype(np.float64, copy=False)
        if llr.shape[1] != self.n_vars:
            raise ValueError(f"llr vector length {llr.shape[1]} != block length {self.n_vars}")
        syn = np.atleast_2d(np.asarray(syndrome))
        if syn.shape != (llr.shape[0], self.n_checks):
            raise ValueError(f"syndrome shape {syn.shape} != ({llr.shape[0]}, {self.n_checks})")
        if syn.dtype not in (np.uint8, np.bool_, np.int8):
            syn = syn.astype(bool)
        syn = np.ascontiguousarray(syn).view(np.uint8)
        st = self._state(llr.shape[0])
        st.set_llr(llr)
        st.set_syndrome(syn)
        st.decode(self._qcfg)
        return st.results()


class _StreamSlot:
    """One device workspace plus pinned result buffers of decode_stream."""

    def __init__(self, plan, batch, precision, engine, n):
        self.state = _native.State(plan, batch, precision)
        self.state.set_engine(engine)
        self.batch = batch
        self.words = _native.PinnedArray((batch, n), np.uint8)
        self.conv = _native.PinnedArray((batch,), np.uint8)
        self.iters = _native.PinnedArray((batch,), np.int64)
        self.inputs = None  # keeps the caller's arrays alive until the copies land


def _stream_decode(self, batches, depth=2, copy=False):
    """Decode an iterable of (llr0, syndrome) batches, yielding (words, converged,
    iterations) per batch in order -- ``decode_batch_arrays`` semantics -- while the
    host<->device copies of one batch overlap the decoding of the next.

    ``depth`` device workspaces are cycled (each ~1.5 GB for 64 codewords of the n=10^6
    code).  Pageable inputs (the reference's float64 arrays) are converted and staged
    into pinned chunks by the library's host threads before ``set_llr`` returns, while
    the previous batch decodes; pinned float32 arrays (``_native.PinnedArray``) are read
    asynchronously and must stay unmodified until their result is yielded.  Yielded
    arrays are views of pinned buffers (kept alive by the views) that are overwritten
    ``depth`` batches later unless ``copy=True``.
    """
    # workspaces persist across calls (per host thread): their whole-decode CUDA graphs
    # are instantiated once
    cache = getattr(self._local, "stream_slots", None)
    if cache is None or len(cache) != max(1, int(depth)):
        cache = self._local.stream_slots = [None] * max(1, int(depth))
    slots, pending = cache, deque()

    def finish(slot):
        slot.state.wait()
        slot.inputs = None
        out = (slot.words.array, slot.conv.array.astype(bool), slot.iters.array)
        return tuple(np.array(a) for a in out) if copy else out

    for i, (llr0, syndrome) in enumerate(batches):
        llr = np.atleast_2d(np.asarray(llr0))
        if llr.dtype != np.float32:
            llr = llr.astype(np.float64, copy=False)
        llr = np.ascontiguousarray(llr)
        if llr.shape[1] != self.n_vars:
            raise ValueError(f"llr vector length {llr.shape[1]} != block length {self.n_vars}")
        syn = np.atleast_2d(np.asarray(syndrome))
        if syn.shape != (llr.shape[0], self.n_checks):
            raise ValueError(f"syndrome shape {syn.shape} != ({llr.shape[0]}, {self.n_checks})")
        syn = np.ascontiguousarray(syn if syn.dtype in (np.uint8, np.bool_, np.int8) else syn.astype(bool)).view(
            np.uint8)
        k = i % len(slots)
        if pending and len(pending) == len(slots):
            yield finish(pending.popleft())
        slot = slots[k]
        if slot is None or slot.batch != llr.shape[0]:
            slot = slots[k] = _StreamSlot(self._plan, llr.shape[0], self.precision, self.engine, self.n_vars)
        st = slot.state
        slot.inputs = (llr, syn)
        st.set_llr(llr)
        st.set_syndrome_hint(syn)  # all-zero check on the library's host threads
        st.decode_async(self._qcfg)
        st.results_async(slot.words.array, slot.conv.array, slot.iters.array)
        pending.append(slot)
    while pending:
        yield finish(pending.popleft())


LayeredDecoder.decode_stream = _stream_decode


def _outcomes(words, converged, iterations):
    return [
        DecodeOutcome(word=words[i], converged=bool(converged[i]), iterations_used=int(iterations[i]))
        for i in range(words.shape[0])
    ]


def decode(llr0, syndrome, index, schedule, cfg, device=0, precision="fp32"):
    """Decode one frame (``decoder.py:444-450``)."""
    dec = LayeredDecoder(index, schedule, cfg, device=device, precision=precision)
    words, converged, iterations = dec.decode_batch_arrays(
        np.asarray(llr0)[None, :], np.asarray(syndrome)[None, :]
    )
    return _outcomes(words, converged, iterations)[0]


def decode_batch(words, index, schedule, cfg, workers=1, device=0, precision="fp32"):
    """Decode a list of (llr0, syndrome) frames (``decoder.py:453-476``).

    Outcomes are in input order and independent of ``workers`` (contiguous chunks on
    host threads sharing one decoder, exactly like the reference).
    """
    if not words:
        return []
    dec = LayeredDecoder(index, schedule, cfg, device=device, precision=precision)
    llr0 = np.stack([np.asarray(w[0], dtype=np.float64) for w in words])
    syndromes = np.stack([np.asarray(w[1]) for w in words])
    if workers <= 1 or len(words) == 1:
        results = [dec.decode_batch_arrays(llr0, syndromes)]
    else:
        chunks = [c for c in np.array_split(np.arange(len(words)), min(workers, len(words))) if c.size]
        with ThreadPoolExecutor(max_workers=len(chunks)) as pool:
            results = list(pool.map(lambda c: dec.decode_batch_arrays(llr0[c], syndromes[c]), chunks))
    out = []
    for triple in results:
        out.extend(_outcomes(*triple))
    return out


class ShardedDecoder:
    """One LayeredDecoder per GPU; a batch is split into contiguous slices.

    Codewords are independent (``SPEC.md:343``), so slice g goes to device g with no
    collective; one host thread per device drives its slice through the C ABI (the
    GIL is released in every call) and outputs are concatenated in order, like
    ``bench._decode_block`` (``bench.py:139-150``).
    """

    def __init__(self, index, schedule, cfg, devices=None, precision="fp32"):
        if devices is None:
            devices = list(range(_native.device_count()))
        if not devices:
            raise RuntimeError("no CUDA device available")
        self.decoders = [LayeredDecoder(index, schedule, cfg, device=d, precision=precision) for d in devices]
        self.n_vars = self.decoders[0].n_vars
        self.n_checks = self.decoders[0].n_checks
        self._pool = ThreadPoolExecutor(max_workers=len(devices))

    def decode_batch_arrays(self, llr0, syndrome):
        llr = np.atleast_2d(np.asarray(llr0))
        syn = np.atleast_2d(np.asarray(syndrome))
        chunks = [c for c in np.array_split(np.arange(llr.shape[0]), len(self.decoders)) if c.size]
        parts = list(
            self._pool.map(
                lambda dc: dc[0].decode_batch_arrays(llr[dc[1]], syn[dc[1]]), zip(self.decoders, chunks)
            )
        )
        return tuple(np.concatenate([p[i] for p in parts]) for i in range(3))


def syndrome_of(word, rows):
    """Syndrome of word(s) under an expanded row adjacency (host utility, ``decoder.py:342-348``).

    Not on the decode path: campaigns that need target syndromes at scale use the
    device encode mode (``qcl_state_set_llr_synthetic(..., encode_mode=1)``).
    """
    word = np.asarray(word)
    bits = np.atleast_2d(word).astype(bool)
    out = np.zeros((bits.shape[0], len(rows)), dtype=np.uint8)
    by_degree = {}
    for i, r in enumerate(rows):
        by_degree.setdefault(len(r), []).append(i)
    for deg, ids in by_degree.items():
        idx = np.stack([np.asarray(rows[i], dtype=np.int64) for i in ids]) if deg else None
        if deg:
            out[:, ids] = np.logical_xor.reduce(bits[:, idx], axis=2)
    return out[0] if word.ndim == 1 else out
