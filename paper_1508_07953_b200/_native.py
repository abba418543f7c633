"""ctypes binding of the C ABI in include/riann_b200.h.

There is no fallback: if the CUDA library is missing, or no B200 is visible,
every compute call raises.  Error codes map onto the reference's exception
types (errors.py:4-17, plus ValueError / IndexError as the reference raises
them).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DimensionError, ModelCapacityError, RiannError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RIANN_LIB") or os.path.join(_PKG, "_lib", "libriann_b200.so")  # RIANN_LIB: development A/B builds

OK, E_VALUE, E_DIMENSION, E_INDEX, E_CAPACITY, E_UNSUPPORTED, E_CUDA, E_STATE = range(8)
F_TEMPORAL, F_DEVICE_PTRS, F_ASYNC, F_KEEP_UNITS = 1, 2, 4, 8


class FrameStatsC(C.Structure):
    _fields_ = [
        ("total_rings", C.c_uint64),
        ("total_distance_evals", C.c_uint64),
        ("sum_cand_final", C.c_uint64),
        ("sum_first_ring", C.c_uint64),
        ("queries", C.c_uint64),
        ("temporal_change", C.c_double),
        ("sum_ring_tests", C.c_uint64),
        ("sum_exact_evals", C.c_uint64),
        ("queries_fallback", C.c_uint64),
    ]


P = C.c_void_p
i32, i64, u32, u64, dbl = C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_double

# name -> (restype, argtypes); every symbol include/riann_b200.h declares
SIGNATURES = {
    "riann_abi_version": (i32, []),
    "riann_debug_checks": (i32, []),
    "riann_last_error": (C.c_char_p, []),
    "riann_ctx_create": (i32, [i32, C.POINTER(P)]),
    "riann_ctx_destroy": (i32, [P]),
    "riann_ctx_stream": (P, [P]),
    "riann_sync": (i32, [P]),
    "riann_ctx_device_bytes": (u64, [P]),
    "riann_ctx_set_path": (i32, [P, i32]),
    "riann_slot_select": (i32, [P, i32]),
    "riann_slot_current": (i32, [P]),
    "riann_slot_free": (i32, [P, i32]),
    "riann_model_set_refs": (i32, [P, P, i64, i32, i32, i32, i32, i32]),
    "riann_model_set_tables": (i32, [P, P, P]),
    "riann_model_build_tables": (i32, [P]),
    "riann_model_get_tables": (i32, [P, i64, i64, P, P]),
    "riann_model_build_table_rows": (i32, [P, i64, i64]),
    "riann_model_table_ptrs": (i32, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(i64), C.POINTER(i64)]),
    "riann_model_attach_shards": (i32, [P, i32, i64, P, P, P]),
    "riann_model_detach_shards": (i32, [P]),
    "riann_process_frame": (i32, [P, P, i32, i32, i32, i32, P, u64, u32, i32, dbl, i32, C.c_uint,
                                  P, P, C.POINTER(FrameStatsC)]),
    "riann_set_prev_units": (i32, [P, P, i64, i32]),
    "riann_field_get": (i32, [P, P, P, i64]),
    "riann_tc_get": (i32, [P, P, i64, C.c_uint]),
    "riann_state_save": (i32, [P]),
    "riann_state_restore": (i32, [P]),
    "riann_timing_enable": (i32, [P, i32]),
    "riann_timing_read": (i32, [P, P, C.POINTER(u64), C.POINTER(u64)]),
    "riann_timing_phases": (i32, [P, P, i32]),
    "riann_timing_phases_frame": (i32, [P, i64, P, i32]),
    "riann_phase_name": (C.c_char_p, [i32]),
    "riann_frame_units": (i32, [P, P, i32, i32, i32, P, P]),
    "riann_normalize_rows": (i32, [P, P, i64, i32, P, P]),
    "riann_normalize_rows_f64": (i32, [P, P, i64, i32, P, P]),
    "riann_one_to_many": (i32, [P, P, P, i64, i32, P]),
    "riann_one_to_many_f64": (i32, [P, P, P, i64, i32, P]),
    "riann_extract_patches": (i32, [P, P, i32, i32, i32, i32, i32, i32, P]),
    "riann_ring_candidates": (i32, [P, i64, dbl, dbl, C.POINTER(i64), C.POINTER(i64), P]),
    "riann_query_batch": (i32, [P, P, P, P, P, i64, i32, dbl, i32, P, P, P, P, P, P, P, P]),
    "riann_exact_nn_batch": (i32, [P, P, i64, P, P]),
    "riann_exact_nn_device": (i32, [P, P, i64, P, P, P]),
    "riann_exact_field": (i32, [P, P, i32, i32, i32, P, P]),
    "riann_field_pack": (i32, [P, P, i64]),
    "riann_apply_effect": (i32, [P, P, i32, i32, P, P, i64, i32, i32, P, P]),
    "riann_pair_dist": (i32, [P, P, P, P, i64, P, P]),
    "riann_init_field": (i32, [i32, i32, i64, P, i32, P]),
    "riann_pairwise_sum": (dbl, [P, i64]),
}

_lib = None
_lock = threading.Lock()       # guards library loading
_ctx_lock = threading.Lock()   # guards the per-device context table


def lib():
    """Load the in-tree CUDA library (built by build.py).  Raises if absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"CUDA library {LIB_PATH} is missing: run `python -m "
                        "paper_1508_07953_b200.build` (there is no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def last_error() -> str:
    return lib().riann_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == E_VALUE:
        raise ValueError(msg)
    if rc == E_DIMENSION:
        raise DimensionError(msg)
    if rc == E_INDEX:
        raise IndexError(msg)
    if rc == E_CAPACITY:
        raise ModelCapacityError(msg)
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RiannError(f"riann_b200 error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def seed_words(seed) -> np.ndarray:
    """numpy SeedSequence entropy coercion for ints / int sequences
    (non-negative ints -> little-endian 32-bit words, [0] for 0)."""
    if isinstance(seed, (bool, np.bool_)):
        raise TypeError("SeedSequence expects int or sequence of ints")
    if isinstance(seed, (int, np.integer)):
        v = int(seed)
        if v < 0:
            raise ValueError("expected non-negative integer")
        if v == 0:
            return np.zeros(1, dtype=np.uint32)
        out = []
        while v > 0:
            out.append(v & 0xFFFFFFFF)
            v >>= 32
        return np.array(out, dtype=np.uint32)
    if isinstance(seed, (float, np.floating)):
        raise TypeError("SeedSequence expects int or sequence of ints")
    parts = [seed_words(v) for v in seed]
    if not parts:
        return np.zeros(0, dtype=np.uint32)
    return np.concatenate(parts).astype(np.uint32)


class Context:
    """One C-ABI context (one CUDA device, one stream) plus the identity of
    the model currently resident on it."""

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(lib().riann_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.model_token = None    # object identity of the resident model (refs + sorted tables)
        self.refs_token = None     # object identity of the model whose refs are resident
        self.model_epoch = 0       # bumped by every model upload (invalidates every slot)
        self.active_slot = 0       # stream slot selected on the C side (riann_slot_select)
        self._next_slot = 1
        self._slot_gen = {0: 0}    # per-slot generation of the device-resident field
        self.lock = threading.RLock()

    # -- stream slots: one device-resident field + prev units per stream ------
    def new_slot(self) -> int:
        with self.lock:
            s = self._next_slot
            self._next_slot += 1
            self._slot_gen[s] = 0
            return s

    def select(self, slot: int) -> None:
        """Make ``slot`` the active stream state (caller holds ``lock``)."""
        if slot != self.active_slot:
            check(lib().riann_slot_select(self.h, int(slot)))
            self.active_slot = slot

    def free_slot(self, slot: int) -> None:
        with self.lock:
            if self.h and slot in self._slot_gen and slot != 0:
                check(lib().riann_slot_free(self.h, int(slot)))
                del self._slot_gen[slot]
                if self.active_slot == slot:
                    self.active_slot = 0

    def advance(self, slot: int) -> tuple:
        """A new field was produced in ``slot``: bump and return its token."""
        self._slot_gen[slot] = self._slot_gen.get(slot, 0) + 1
        return self.token(slot)

    def token(self, slot: int) -> tuple:
        """Identity of the field currently resident in ``slot``."""
        return (id(self), slot, self.model_epoch, self._slot_gen.get(slot, -1))

    @property
    def stream(self) -> int:
        return int(lib().riann_ctx_stream(self.h) or 0)

    def close(self):
        if self.h:
            lib().riann_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}
_default_device = None


def set_device(device: int) -> None:
    """Select the GPU the package's module-level API runs on."""
    global _default_device
    _default_device = int(device)


def current_device() -> int:
    if _default_device is not None:
        return _default_device
    return int(os.environ.get("LOCAL_RANK", "0"))


def context(device: int | None = None) -> Context:
    d = current_device() if device is None else int(device)
    ctx = _contexts.get(d)
    if ctx is None:
        with _ctx_lock:
            ctx = _contexts.get(d)
            if ctx is None:
                ctx = Context(d)
                _contexts[d] = ctx
    return ctx


def set_frame_path(path: int, device: int | None = None) -> None:
    """Path mask: 0 = auto (anchor-grouped frame phases, tensor-core exact
    comparator where supported); 1 = per-query frame kernel only; 2 = SIMT
    exact comparator.  Results are identical; this exists for testing and
    measurement."""
    ctx = context(device)
    with ctx.lock:
        check(lib().riann_ctx_set_path(ctx.h, int(path)))
