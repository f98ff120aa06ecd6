"""Single-process multi-GPU fan-out of the select path (SURVEY.md §8(b) Threading, §8(e)).

The reference engine is one single-threaded process (configurator.py:368-373).  A drop-in that
wants every GPU of the box cannot rely on one process per GPU, so the fan-out lives inside the
library (include/slackpipe_b200.h ``sp_group_*``): ``DeviceGroup`` owns one context per device,
``GroupOpTable`` is an ``OpTable`` replicated on every member (mutations go to every replica in
the same order, so the replicas stay bit-identical), and ``GroupOpTable.select_batch`` splits a
host batch into contiguous shards, one per device, all in flight at once, decisions written in
global invocation order into the caller's arrays — the same result as ``OpTable.select_batch``
on one GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, load_library, ptr
from .configurator import OpTable, SelectResult


class _MemberContext:
    """A group member's context, shaped like ``_lib.Context`` for code that takes one."""

    def __init__(self, lib, handle, device):
        self.lib = lib
        self.handle = handle
        self.device = device

    def synchronize(self) -> None:
        check(self.lib.sp_ctx_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        return int(self.lib.sp_ctx_launch_count(self.handle))


class DeviceGroup:
    """One library context per listed CUDA device (devices may repeat: independent contexts on
    one GPU).  ``devices=None`` takes every visible device."""

    def __init__(self, devices: Sequence[int] | None = None):
        self.lib = load_library()
        if devices is None:
            import torch

            devices = list(range(torch.cuda.device_count()))
        devs = np.ascontiguousarray(list(devices), dtype=np.int32)
        if len(devs) < 1:
            raise ValueError("DeviceGroup: no devices")
        h = C.c_void_p()
        check(self.lib.sp_group_create(len(devs), ptr(devs), C.byref(h)), "sp_group_create")
        self.handle = h
        self.devices = [int(d) for d in devs]
        self.members = []
        for i in range(len(devs)):
            ch = C.c_void_p()
            d = C.c_int32()
            check(self.lib.sp_group_member(self.handle, i, C.byref(ch), C.byref(d)))
            self.members.append(_MemberContext(self.lib, ch, int(d.value)))

    def __len__(self) -> int:
        return len(self.devices)

    @property
    def launch_count(self) -> int:
        return int(self.lib.sp_group_launch_count(self.handle))

    def table(self, spec, scenario, *, kinds: Sequence[str] | None = None) -> "GroupOpTable":
        return GroupOpTable(spec, scenario, group=self, kinds=kinds)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.sp_group_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class GroupOpTable(OpTable):
    """``OpTable`` (configurator.py:159-318) replicated on every device of a ``DeviceGroup``.
    Host arrays (``lat`` etc.) are the reference's; the single-invocation reference methods
    (``select``, ``affinity``) run on member 0, batched ``select_batch`` fans out."""

    def __init__(self, spec, scenario, *, group: DeviceGroup, kinds: Sequence[str] | None = None):
        self._group = group
        super().__init__(spec, scenario, kinds=kinds)

    def _create_device(self, device) -> None:
        g = self._group
        self._ctx = g.members[0]
        n, lat, lat_init, res, batch32, pool, price, gkind, rank32 = self._device_columns()
        h = C.c_void_p()
        check(g.lib.sp_group_table_create(
            g.handle, n, ptr(lat), ptr(lat_init), ptr(res), ptr(batch32), ptr(pool), ptr(price),
            ptr(gkind), ptr(rank32), len(self.global_kinds), self.ref_index, C.byref(h)),
            "sp_group_table_create")
        self._ghandle = h
        r0 = C.c_void_p()
        check(g.lib.sp_group_table_replica(self._ghandle, 0, C.byref(r0)))
        self._handle = r0  # member 0's replica backs the single-invocation reference API

    def replica(self, i: int) -> C.c_void_p:
        r = C.c_void_p()
        check(self._group.lib.sp_group_table_replica(self._ghandle, int(i), C.byref(r)))
        return r

    def replica_latency(self, i: int) -> np.ndarray:
        out = np.empty_like(self.lat)
        check(self._group.lib.sp_group_table_get_latency(self._group.handle, self._ghandle, int(i),
                                                         ptr(out)))
        return out

    def close(self) -> None:
        if getattr(self, "_ghandle", None):
            self._group.lib.sp_group_table_destroy(self._group.handle, self._ghandle)
            self._ghandle = None
            self._handle = None

    def set_latency(self, index: int, latency_s: float) -> None:
        """configurator.py:211-213 on every replica."""
        i = np.array([index], dtype=np.int32)
        v = np.array([latency_s], dtype=np.float64)
        check(self._group.lib.sp_group_table_set_latency(self._group.handle, self._ghandle, 1,
                                                         ptr(i), ptr(v)))
        self.entries[index].latency_s = latency_s
        self.lat[index] = latency_s

    def select_batch(self, slack, alpha, available, *, upstream_supply, min_batch, flags,
                     kind_min: bool = False, mode: str = "auto", out: dict | None = None) -> SelectResult:
        return group_select_batch([self], slack, alpha, available, upstream_supply=upstream_supply,
                                  min_batch=min_batch, flags=flags, kind_min=kind_min, mode=mode,
                                  out=out)

    def fold(self, idx, obs, *, beta: float = 0.5, dfp_count: int = 10, dfp_on: bool = True,
             fb_frozen: bool = False) -> None:
        """sp_feedback_fold of one host observation stream into every replica, then the host
        mirror is refreshed from member 0."""
        group_fold([self], None, idx, obs, beta=beta, dfp_count=dfp_count, dfp_on=dfp_on,
                   fb_frozen=fb_frozen)


def _host(a, dtype, shape, name):
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.shape != shape:
        raise ValueError(f"{name} must have shape {shape}")
    return a


def group_select_batch(tables: Sequence[GroupOpTable], slack, alpha: float, available, *,
                       upstream_supply, min_batch, flags, op=None, kind_min: bool = False,
                       mode: str = "auto", out: dict | None = None) -> SelectResult:
    """``select_batch`` (configurator.py:239-300 over N invocations) with host numpy buffers,
    sharded over the group's devices.  Pinned (page-locked, mapped) buffers let every device
    read and write its shard over PCIe in one launch."""
    if not tables:
        raise ValueError("select_batch: no tables")
    g = tables[0]._group
    K = tables[0].K
    slack = np.asarray(slack)
    N = int(slack.shape[0])
    slack = _host(slack, np.float64, (N, K), "slack")
    available = _host(available, np.int32, (N,), "available")
    upstream_supply = _host(upstream_supply, np.int32, (N,), "upstream_supply")
    min_batch = _host(min_batch, np.int32, (N,), "min_batch")
    flags = _host(flags, np.uint32, (N,), "flags")
    if op is not None:
        op = _host(op, np.int32, (N,), "op")
    if out is None:
        out = {"idx": np.empty(N, np.int32), "code": np.empty(N, np.int32),
               "fill": np.empty(N, np.int32), "obj": np.empty(N), "slack": np.empty(N),
               "wait": np.empty(N)}
        if kind_min:
            out["kind_min"] = np.empty((N, K))
    arr = (C.c_void_p * len(tables))(*[t._ghandle.value for t in tables])
    check(g.lib.sp_group_select_batch(
        g.handle, len(tables), C.cast(arr, C.c_void_p), float(alpha), N, ptr(op), ptr(slack),
        ptr(available), ptr(upstream_supply), ptr(min_batch), ptr(flags), ptr(out["idx"]),
        ptr(out["code"]), ptr(out.get("fill")), ptr(out.get("obj")), ptr(out.get("slack")),
        ptr(out.get("wait")), ptr(out.get("kind_min") if kind_min else None), _lib.MODES[mode]),
        "sp_group_select_batch")
    return SelectResult(out)


def group_fold(tables: Sequence[GroupOpTable], op, idx, obs, *, beta: float = 0.5,
               dfp_count: int = 10, dfp_on: bool = True, fb_frozen: bool = False) -> None:
    """fold_observations (manager.py:436-457) into every replica of the group tables."""
    g = tables[0]._group
    n = int(np.asarray(obs).shape[0])
    idx = _host(idx, np.int32, (n,), "idx")
    obs = _host(obs, np.float64, (n,), "obs")
    if op is not None:
        op = _host(op, np.int32, (n,), "op")
    arr = (C.c_void_p * len(tables))(*[t._ghandle.value for t in tables])
    check(g.lib.sp_group_feedback_fold(g.handle, len(tables), C.cast(arr, C.c_void_p), n, ptr(op),
                                       ptr(idx), ptr(obs), float(beta), int(dfp_count),
                                       1 if dfp_on else 0, 1 if fb_frozen else 0),
          "sp_group_feedback_fold")
    for t in tables:
        t.sync_from_device()
