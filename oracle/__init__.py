"""CPU oracle for the configurator hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithm (`slackpipe`, /root/reference/pkg/src/slackpipe)
on the CPU, function by function, each citing the reference file:line it follows.  It is the
checker, never the product: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
``paper_2102_01887_b200`` never imports it and fails loudly without its CUDA library.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``, run in the
build container where /root/reference is importable) and, when the reference is importable,
against the reference itself on fresh random inputs.

Modules
  optable   OpTable.__init__/scores/_argmin/select/affinity  (configurator.py:159-318)
  slack     compute_slack / Configurator.slack_by_kind, path decomposition, forward-DP
            restatement for DAGs whose paths cannot be enumerated (configurator.py:64-106,
            493-543; pipeline.py:428-451)
  feedback  apply_feedback + PipelineRun._apply_feedback + recalibrate_unobserved
            (manager.py:45-47, 436-457; configurator.py:463-491)
  queueing  estimate_queueing / queueing_by_kind ordered sums (configurator.py:109-119, 511-524)
  cselect   ctypes loader of select_oracle.c, a scalar C restatement of OpTable.select used for
            full-size (2^20 invocations) parity checks in seconds
"""
