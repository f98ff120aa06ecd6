"""CPU restatement of the feedback fold — TEST ORACLE ONLY.

Follows PipelineRun._apply_feedback (manager.py:436-457) with apply_feedback
(manager.py:45-47), FeedbackStore.observe (manager.py:99-101) and
Configurator.recalibrate_unobserved (configurator.py:470-491), one observation at a time.
State per table: lat (live), lat_init, ref_index, completed_ref, obs_count per entry.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def apply_feedback(old: float, obs: float, beta: float) -> float:
    return beta * obs + (1.0 - beta) * old


@dataclass
class FoldState:
    lat: np.ndarray
    lat_init: np.ndarray
    ref_index: int
    completed_ref: int = 0
    obs_count: np.ndarray | None = None

    def __post_init__(self):
        if self.obs_count is None:
            self.obs_count = np.zeros(len(self.lat), dtype=np.int64)


def fold(states, op, idx, obs, *, beta=0.5, dfp_count=10, dfp_on=True, fb_frozen=False):
    """Sequential fold of observations in completion order (mutates states)."""
    for j in range(len(idx)):
        st = states[0 if op is None else int(op[j])]
        e = int(idx[j])
        if e == st.ref_index:
            st.completed_ref += 1
        st.obs_count[e] += 1
        if fb_frozen:
            continue
        st.lat[e] = apply_feedback(float(st.lat[e]), float(obs[j]), beta)
        if e == st.ref_index and st.completed_ref == dfp_count and dfp_on:
            if st.ref_index >= 0:
                init_ref = float(st.lat_init[st.ref_index])
                if init_ref > 0.0:
                    ratio = float(st.lat[st.ref_index]) / init_ref
                    for i in range(len(st.lat)):
                        if i == st.ref_index or st.obs_count[i] > 0:
                            continue
                        st.lat[i] = float(st.lat_init[i]) * ratio
    return states
