"""ctypes binding of libslackpipe_b200.so (C-ABI declared in include/slackpipe_b200.h).

The library is the ONLY compute path of this package: there is no CPU fallback.  If the
shared object is missing or no B200 is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libslackpipe_b200.so"

SP_OK = 0
SP_E_INVALID = -1
SP_E_CUDA = -2
SP_E_NOMEM = -3
SP_E_UNSUPPORTED = -4
SP_E_RUNTIME = -5

SP_MEM_HOST = 0
SP_MEM_DEVICE = 1

SP_DEC_NONE = 0
SP_DEC_ASSIGN = 1
SP_DEC_DELAY = 2
SP_DEC_FEASIBLE = 4
SP_DEC_ERROR = 3  # the reference raises ValueError (NaN scores leave no tie)

SP_FLAG_ALLOW_DELAY = 1
SP_FLAG_EXCL_SHIFT = 8

SP_MODE_AUTO = 0
SP_MODE_PLAN = 1
SP_MODE_SCAN = 2
MODES = {"auto": SP_MODE_AUTO, "plan": SP_MODE_PLAN, "scan": SP_MODE_SCAN}

SP_HEAD_PRESENT = 1
SP_HEAD_FORCED = 2
SP_SPEC_SDB = 1
SP_SPEC_FORCED = 2
SP_SPEC_HOLD_EXPIRED = 4
SP_COMMIT_FIFO = 1
SP_COMMIT_ESLC = 2

MAX_KINDS = 24          # table kinds (SP_MAX_KINDS); the staircase plan takes <= 8

# (name, restype, argtypes) for every exported symbol; the CPU test suite checks that
# the shared object exports exactly what include/slackpipe_b200.h declares.
_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_d = C.c_double
_pp = C.POINTER(C.c_void_p)
SIGNATURES = {
    "sp_version": (C.c_int, []),
    "sp_ctx_create": (C.c_int, [C.c_int, _pp]),
    "sp_ctx_destroy": (C.c_int, [_p]),
    "sp_ctx_set_stream": (C.c_int, [_p, _p]),
    "sp_ctx_synchronize": (C.c_int, [_p]),
    "sp_ctx_set_option": (C.c_int, [_p, C.c_char_p, _i64]),
    "sp_last_error": (C.c_char_p, [_p]),
    "sp_ctx_launch_count": (_i64, [_p]),
    "sp_table_create": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _i32, _pp]),
    "sp_table_destroy": (C.c_int, [_p, _p]),
    "sp_table_set_latency": (C.c_int, [_p, _p, _i32, _p, _p]),
    "sp_table_get_latency": (C.c_int, [_p, _p, _p]),
    "sp_table_prepare": (C.c_int, [_p, _p, _d]),
    "sp_table_invalidate": (C.c_int, [_p, _p]),
    "sp_table_prepare_many": (C.c_int, [_p, _p, _i32, _p]),
    "sp_table_plan_supported": (C.c_int, [_p]),
    "sp_table_plan_bytes": (C.c_int, [_p, _p, _d, C.POINTER(_i64)]),
    "sp_table_plan_image": (C.c_int, [_p, _p, _d, _i32, _p, _i64, C.POINTER(_i64)]),
    "sp_scores": (C.c_int, [_p, _p, _p, _d, _p, _p]),
    "sp_select_batch": (C.c_int, [_p, _i32, _p, _d, _i32, _p, _p, _p, _p, _p, _p,
                                  _p, _p, _p, _p, _p, _p, _p, _i32, _i32]),
    "sp_affinity_from_minima": (C.c_int, [_p, _i32, _i32, _p, _p, _p, _p, _i32]),
    "sp_affinity_batch": (C.c_int, [_p, _i32, _p, _d, _i32, _p, _p, _p, _p, _i32]),
    "sp_dag_create": (C.c_int, [_p, _i32, _p, _p, _p, _p, _i32, _p, _pp]),
    "sp_dag_destroy": (C.c_int, [_p, _p]),
    "sp_slack_batch": (C.c_int, [_p, _p, _i32, _p, _i32, _p, _p, _i32, _p, _p, _p, _i32]),
    "sp_queueing": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p]),
    "sp_feedback_fold": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _p, _d, _i32, _i32, _i32, _i32]),
    "sp_table_get_counters": (C.c_int, [_p, _p, _p, _p]),
    "sp_table_set_counters": (C.c_int, [_p, _p, _i32, _p]),
    "sp_speculate_batch": (C.c_int, [_p, _i32, _p, _d, _i32, _p, _i32] + [_p] * 21 + [_i32]),
    "sp_commit_round": (C.c_int, [_p, _i32, _i32, _p, _d] + [_p] * 10 + [_i32] + [_p] * 6 + [_i32]),
    "sp_observation_quantiles": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _p, _d, _d, _p, _p, _p, _i32]),
    "sp_slack_select_batch": (C.c_int, [_p, _p, _i32, _p, _d, _i32, _p, _i32, _p, _p, _i32, _p]
                              + [_p] * 11 + [_i32]),
    "sp_simulate_observations": (C.c_int, [_p, _i32] + [_p] * 8),
    "sp_profile_configs": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _p, _p,
                                     _i32, _p, _p, _i64, _p, _p, _p, _p]),
    "sp_pow_correctly_rounded": (C.c_int, [_p, _i32, _p, _p, _p]),
    "sp_simulate_and_fold": (C.c_int, [_p, _p, _i32, _p, _p, _p, _p, _p, _p, _d, _i32, _i32, _i32, _p, _p]),
    "sp_des_create": (C.c_int, [_p, _p, _pp]),
    "sp_des_destroy": (C.c_int, [_p, _p]),
    "sp_des_prepare": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _i32, _i32]),
    "sp_des_set_capacity": (C.c_int, [_p, _d]),
    "sp_des_set_mode": (C.c_int, [_p, _i32]),
    "sp_des_arena_bytes": (_i64, [_p]),
    "sp_des_draws": (C.c_int, [_i32, _p, _i32, _d, _d, _d, _p, _p]),
    "sp_des_run": (C.c_int, [_p, _p, _i32, _i32, _p, _p, _p, _p, _i32, _p, _p, _i32, _p, _p, _p, _i32,
                             _p, _i32]),
    "sp_group_create": (C.c_int, [_i32, _p, _pp]),
    "sp_group_destroy": (C.c_int, [_p]),
    "sp_group_size": (_i32, [_p]),
    "sp_group_member": (C.c_int, [_p, _i32, _pp, _p]),
    "sp_group_launch_count": (_i64, [_p]),
    "sp_group_table_create": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _i32, _pp]),
    "sp_group_table_destroy": (C.c_int, [_p, _p]),
    "sp_group_table_replica": (C.c_int, [_p, _i32, _pp]),
    "sp_group_table_set_latency": (C.c_int, [_p, _p, _i32, _p, _p]),
    "sp_group_table_get_latency": (C.c_int, [_p, _p, _i32, _p]),
    "sp_group_select_batch": (C.c_int, [_p, _i32, _p, _d, _i32, _p, _p, _p, _p, _p, _p,
                                        _p, _p, _p, _p, _p, _p, _p, _i32]),
    "sp_group_feedback_fold": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _p, _d, _i32, _i32, _i32]),
}


class SlackpipeError(RuntimeError):
    """CUDA / unsupported-configuration failure inside libslackpipe_b200."""


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None):
    """dlopen the library and bind every signature (no GPU needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise SlackpipeError(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load_library().sp_last_error(None)
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == SP_OK:
        return
    msg = last_error()
    if rc == SP_E_INVALID:
        raise ValueError(msg)
    if rc == SP_E_RUNTIME:
        raise RuntimeError(msg)
    raise SlackpipeError(f"{what}: {msg} (code {rc})" if what else f"{msg} (code {rc})")


class Context:
    """One CUDA device + stream owned by the library (sp_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        check(self.lib.sp_ctx_create(int(device), C.byref(h)), "sp_ctx_create")
        self.handle = h
        self.device = int(device)

    def set_stream(self, stream_handle: int) -> None:
        check(self.lib.sp_ctx_set_stream(self.handle, C.c_void_p(int(stream_handle))))

    def synchronize(self) -> None:
        check(self.lib.sp_ctx_synchronize(self.handle))

    def set_option(self, name: str, value: int) -> None:
        """Dispatch variant of this context (tests / tools; the environment is read once, at
        creation)."""
        check(self.lib.sp_ctx_set_option(self.handle, name.encode(), int(value)))

    @property
    def launch_count(self) -> int:
        return int(self.lib.sp_ctx_launch_count(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.sp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


_ctx: dict[int, Context] = {}


def default_device() -> int:
    env = os.environ.get("SLACKPIPE_B200_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def get_context(device: int | None = None) -> Context:
    d = default_device() if device is None else int(device)
    with _lib_lock:
        c = _ctx.get(d)
    if c is None:
        c = Context(d)
        with _lib_lock:
            _ctx[d] = c
    return c


def ptr(a):
    """Data pointer of a torch tensor (device or host) or a numpy array (host), as an int
    (ctypes passes it as void*; None is NULL)."""
    if a is None:
        return None
    dp = getattr(a, "data_ptr", None)
    if dp is not None:
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return dp()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported buffer type {type(a)!r}")
