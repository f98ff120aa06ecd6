"""The speculation drop-in's host bookkeeping, end to end on the CPU (build container only).

``speculate_from_buffer(conf, op, buffer)`` takes its decisions from one sp_speculate_batch call
and replays the reference's bookkeeping (invocations, queues, holds, wake-ups, forced counts,
decision log).  Here the unmodified reference engine runs the AMBER scenario with its
``Configurator.speculate_from_buffer`` replaced by the drop-in, and the device call replaced by
the oracle restatement (oracle/speculate.py, itself pinned to 15,000 recorded calls) over the
engine's live tables — so the run's decision log and CSV row must equal the reference's own
golden run (15,290 decision-log rows at the 50 % target).  The device side of
the same call is covered bit-for-bit by tests/test_gpu_speculate.py.
"""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from oracle import optable
from oracle import speculate as osp

BUNDLE = Path("/root/reference/pkg/scenarios/branching")


def _oracle_tables(conf):
    kinds = list(conf.kinds)
    out = []
    for name, t in conf.tables.items():
        gk = [kinds.index(e.backend_kind) for e in t.entries]
        out.append(optable.from_columns(lat=np.array(t.lat, dtype=np.float64), res=t.res, batch=t.batch,
                                        pool=t.pool, price=t.price, gkind=gk, id_rank=t.id_rank,
                                        n_kinds=len(kinds), ref_index=t.ref_index))
    return out


def _fake_batch(conf_box):
    """speculate_batch stand-in: the oracle over the live reference tables."""
    def run(tables, alpha, pool, op, n_buf, supply, now, target, rmin, rmax, slack0, flags, w_ptr,
            w_tab, w_eidx, w_count, **_):
        conf = conf_box[0]
        otabs = _oracle_tables(conf)
        K = len(pool)
        sq = [[] for _ in range(K)]
        cq = [[] for _ in range(K)]
        for q, lists in enumerate((sq, cq)):
            for k in range(K):
                for w in range(w_ptr[q * K + k], w_ptr[q * K + k + 1]):
                    lists[k].append([int(w_tab[w]), int(w_eidx[w]), int(w_count[w])])
        dec, delay = osp.speculate(otabs, int(op[0]), int(n_buf[0]), int(supply[0]), float(now[0]),
                                   float(target[0]), float(rmin[0]), float(rmax[0]), pool, alpha,
                                   int(flags[0]), sq, cq, slack0[0])
        n = len(dec)
        return {"off": np.array([0, n]), "idx": np.array([d[0] for d in dec], np.int64),
                "fill": np.array([d[1] for d in dec], np.int64),
                "slack": np.array([d[2] for d in dec]), "obj": np.array([d[3] for d in dec]),
                "n": np.array([n]), "delay_idx": np.array([delay[0] if delay else -1]),
                "delay_wait": np.array([delay[1] if delay else 0.0])}
    return run


def test_speculate_dropin_reproduces_the_reference_run(ref, monkeypatch, tmp_path):
    from slackpipe import cli, configurator

    import paper_2102_01887_b200.speculate as dropin

    box = [None]
    monkeypatch.setattr(dropin, "speculate_batch", _fake_batch(box))

    def spec(self, op, buffer):
        box[0] = self
        return dropin.speculate_from_buffer(self, op, buffer)

    monkeypatch.setattr(configurator.Configurator, "speculate_from_buffer", spec)
    out = tmp_path / "run.csv"
    log = tmp_path / "decisions.tsv"
    rc = cli.main(["run", "--pipeline", str(BUNDLE / "pipeline.json"), "--scenario",
                   str(BUNDLE / "scenario.json"), "--trace", str(BUNDLE / "trace.jsonl"),
                   "--target", "142.20064921472454", "--metadata-dir", str(tmp_path / "md"),
                   "--report", str(out), "--decision-log", str(log)])
    assert rc == 0
    row = out.read_text().strip().splitlines()[-1].split(",")
    # golden CSV row of the reference's own run
    assert row[1:] == ["142.20064921472454", "132.73451153109434", "0.9334311218977895",
                       "0.16671542613566986", "1.0", "20", "0", "0"]
    assert len(log.read_text().strip().splitlines()) == 1 + 15290  # header + decisions
    digest = hashlib.sha256(log.read_bytes()).hexdigest()[:16]
    assert digest == "4647eeb560b36a71"


def test_speculate_and_commit_dropins_reproduce_the_reference_run(ref, monkeypatch, tmp_path):
    """Both Configurator hot loops replaced — speculate_from_buffer and pump_commits — with the
    device calls stood in by the pinned oracles (oracle/speculate.py, oracle/commit.py): the
    reference engine's golden AMBER run is reproduced exactly."""
    from slackpipe import cli, configurator

    import paper_2102_01887_b200.commit as cdrop
    import paper_2102_01887_b200.speculate as dropin
    from oracle import commit as oc

    box = [None]
    monkeypatch.setattr(dropin, "speculate_batch", _fake_batch(box))

    def fake_candidates(tables, slacks, heads, buffered, depths, full_kinds, alpha, ablations=()):
        conf = box[0]
        kinds = list(conf.kinds)
        otabs = _oracle_tables(conf)
        full = sum(1 << kinds.index(k) for k in full_kinds)
        sl = [np.array([s[k] for k in kinds]) if s is not None else None for s in slacks]
        hs = [oc.Head(h.fill, h.forced, h.invocation_id, h.spec_eidx, h.spec_slack_s, h.spec_objective)
              if h is not None else None for h in heads]
        w = oc.round_winner(otabs, sl, hs, full, buffered, depths, alpha, fifo="pbc" in ablations,
                            eslc="eslc" in ablations)
        if w is None:
            return None
        j, (e, fill, s_k, obj) = w
        return (j, tables[j].entries[e], e, fill, s_k, obj)

    monkeypatch.setattr(cdrop, "commit_candidates", fake_candidates)

    def spec(self, op, buffer):
        box[0] = self
        return dropin.speculate_from_buffer(self, op, buffer)

    def pump(self, buffered_count, topup):
        box[0] = self
        return cdrop.pump_commits(self, buffered_count, topup)

    monkeypatch.setattr(configurator.Configurator, "speculate_from_buffer", spec)
    monkeypatch.setattr(configurator.Configurator, "pump_commits", pump)
    out = tmp_path / "run.csv"
    log = tmp_path / "decisions.tsv"
    rc = cli.main(["run", "--pipeline", str(BUNDLE / "pipeline.json"), "--scenario",
                   str(BUNDLE / "scenario.json"), "--trace", str(BUNDLE / "trace.jsonl"),
                   "--target", "142.20064921472454", "--metadata-dir", str(tmp_path / "md"),
                   "--report", str(out), "--decision-log", str(log)])
    assert rc == 0
    row = out.read_text().strip().splitlines()[-1].split(",")
    assert row[1:] == ["142.20064921472454", "132.73451153109434", "0.9334311218977895",
                       "0.16671542613566986", "1.0", "20", "0", "0"]
    assert hashlib.sha256(log.read_bytes()).hexdigest()[:16] == "4647eeb560b36a71"


import pytest


def _cli_run(cli, tmp, name, extra):
    out = tmp / f"{name}.csv"
    log = tmp / f"{name}.tsv"
    rc = cli.main(["run", "--pipeline", str(BUNDLE / "pipeline.json"), "--scenario",
                   str(BUNDLE / "scenario.json"), "--trace", str(BUNDLE / "trace.jsonl"),
                   "--target", "142.20064921472454", "--metadata-dir", str(tmp / f"md_{name}"),
                   "--report", str(out), "--decision-log", str(log), *extra])
    assert rc == 0
    return out.read_text().strip().splitlines()[-1].split(",")[1:], log.read_bytes()


@pytest.mark.parametrize("extra", [["--ablate", "eslc"], ["--ablate", "pbc"], ["--ablate", "fb"],
                                   ["--ablate", "eslc,pbc"], ["--failure-rate", "0.05"]],
                         ids=["eslc", "pbc", "fb", "eslc+pbc", "failures"])
def test_dropins_under_ablations_and_failures(ref, monkeypatch, tmp_path, extra):
    """Both drop-ins under the eslc / pbc / fb ablations and with invocation failures (retries
    re-enter through speculate_fixed): the run's CSV row and decision log equal the unmodified
    reference's own run with the same flags, byte for byte — which also pins that the drop-ins
    evaluate slack_by_kind exactly where the reference does (its per-version cache)."""
    from slackpipe import cli, configurator

    import paper_2102_01887_b200.commit as cdrop
    import paper_2102_01887_b200.speculate as dropin

    want_row, want_log = _cli_run(cli, tmp_path, "ref", extra)
    box = [None]
    monkeypatch.setattr(dropin, "speculate_batch", _fake_batch(box))
    from oracle import commit as oc

    def fake_candidates(tables, slacks, heads, buffered, depths, full_kinds, alpha, ablations=()):
        conf = box[0]
        kinds = list(conf.kinds)
        otabs = _oracle_tables(conf)
        full = sum(1 << kinds.index(k) for k in full_kinds)
        sl = [np.array([s[k] for k in kinds]) if s is not None else None for s in slacks]
        hs = [oc.Head(h.fill, h.forced, h.invocation_id, h.spec_eidx, h.spec_slack_s, h.spec_objective)
              if h is not None else None for h in heads]
        w = oc.round_winner(otabs, sl, hs, full, buffered, depths, alpha, fifo="pbc" in ablations,
                            eslc="eslc" in ablations)
        if w is None:
            return None
        j, (e, fill, s_k, obj) = w
        return (j, tables[j].entries[e], e, fill, s_k, obj)

    monkeypatch.setattr(cdrop, "commit_candidates", fake_candidates)

    def spec(self, op, buffer):
        box[0] = self
        return dropin.speculate_from_buffer(self, op, buffer)

    def pump(self, buffered_count, topup):
        box[0] = self
        return cdrop.pump_commits(self, buffered_count, topup)

    monkeypatch.setattr(configurator.Configurator, "speculate_from_buffer", spec)
    monkeypatch.setattr(configurator.Configurator, "pump_commits", pump)
    row, log = _cli_run(cli, tmp_path, "dropin", extra)
    assert row == want_row
    assert log == want_log
