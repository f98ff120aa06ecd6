"""B200-native configuration-optimizer hot path of Llama (arXiv 2102.01887, ref. pkg `slackpipe`).

Drop-in for the reference's configurator path: ``OpTable`` / ``select_config`` /
``affinity`` / ``compute_slack`` / ``estimate_queueing`` / ``objective`` /
``apply_feedback`` keep the reference's names and semantics; batched entry points
(``select_batch``, ``SlackGraph.slack_batch``, ``fold_observations``) run the same
functions over millions of invocations on sm_100a kernels in libslackpipe_b200.so.
"""
from ._lib import SlackpipeError, get_context, load_library
from .configurator import (
    ABLATION_TOKENS,
    AffinityScore,
    Decision,
    OpTable,
    RawTable,
    SelectResult,
    Slack,
    TuningParams,
    affinity,
    affinity_from_minima,
    estimate_queueing,
    make_flags,
    objective,
    remaining_path_latency,
    select_batch,
    select_config,
)
from . import metadata
from .commit import commit_candidates, commit_round, pump_commits
from .group import DeviceGroup, GroupOpTable, group_fold, group_select_batch
from .feedback import apply_feedback, fold_observations, observation_quantiles, set_table_counters, simulate_and_fold, simulate_observations, table_counters
from .pipeline import (ConfigAssignment, ConfigEntry, ConfigSpec, Knob, KnobTemplate, OperationSpec, PipelineDag,
                       enumerate_configs, reference_config)
from .profiler import profile_operation
from .scenario import BackendSpec, GroundTruthModel, OpKindTruth, Scenario
from .slack import SlackGraph, compute_slack
from .speculate import speculate_batch, speculate_from_buffer

__version__ = "0.1.0"

__all__ = [
    "ABLATION_TOKENS", "AffinityScore", "BackendSpec", "DeviceGroup", "GroupOpTable",
    "group_fold", "group_select_batch", "ConfigEntry", "ConfigSpec", "Decision",
    "OpTable", "PipelineDag", "RawTable", "Scenario", "SelectResult", "Slack", "SlackGraph",
    "SlackpipeError", "TuningParams", "affinity", "affinity_from_minima", "apply_feedback",
    "commit_candidates", "commit_round", "compute_slack", "estimate_queueing", "fold_observations", "get_context", "load_library",
    "make_flags", "metadata", "objective", "pump_commits", "observation_quantiles", "reference_config", "remaining_path_latency", "select_batch",
    "select_config", "set_table_counters", "simulate_and_fold", "simulate_observations", "speculate_batch", "speculate_from_buffer",
    "table_counters", "ConfigAssignment", "Knob", "KnobTemplate", "OperationSpec", "enumerate_configs",
    "profile_operation", "GroundTruthModel", "OpKindTruth",
]
