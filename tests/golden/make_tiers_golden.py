"""Dump tier-driven scale-out fixtures from the reference SIMULATOR itself
(run HERE only; the GPU box never runs this file).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_tiers_golden.py

For each case the unmodified reference simulator (``simengine.run``, strategy
lambda_scale) serves a burst that triggers scale-outs; ``compose_schedule``
as seen by ``simengine`` is wrapped to record the sub-groups it was given and
the schedule lines it returned, and the ``scale_out`` events give the demand
nodes, their hot/warm/cold classes and the startup sources.  Together with the
initial residency this pins ``scaleout.plan_from_tiers`` (startup_plan ->
_warm_and_hot -> _launch_lambda_scale, simengine.py:442-467, :507-521,
:564-590) to the reference's own behaviour.  Writes tiers.json.
"""
from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from blockcast import simengine as S  # noqa: E402
from blockcast.multicast import ModelSpec, schedule_to_lines  # noqa: E402
from blockcast.workload import TraceRecord  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GB = 10 ** 9

# (label, node_count, initial_gpu, initial_memory, k, b, burst)
CASES = [
    ("gpu0_k1", 8, [0], [0], 1, 8, 60),
    ("gpu0_host7_k2", 8, [0], [7], 2, 8, 60),
    ("host_only_k1", 8, [], [3], 1, 8, 60),
    ("host_only_k2", 8, [], [3], 2, 8, 60),
    ("gpu01_host7_k3", 8, [0, 1], [7], 3, 8, 80),
    ("gpu0_warm_k2", 6, [0], [0, 2, 4], 2, 4, 40),
    ("ssd_bootstrap", 5, [], [], 1, 4, 30),
]


def run_case(label, n, gpu, mem, k, b, burst):
    cluster = S.ClusterSpec(node_count=n)
    model = ModelSpec("m0", 16 * GB, 32)
    calls = []
    real = S.compose_schedule

    def spy(groups, plan, *a, **kw):
        sched = real(groups, plan, *a, **kw)
        calls.append({"groups": [{"source": g.source, "members": list(g.member_nodes),
                                  "order": list(g.transfer_order)} for g in groups],
                      "lines": schedule_to_lines(sched)})
        return sched
    S.compose_schedule = spy
    try:
        trace = [TraceRecord(f"r{i}", 0.0, "m0", 128, 32) for i in range(burst)]
        res = S.run(cluster, [model], "lambda_scale", trace, S.AutoscalePolicy(), k=k, block_count=b,
                    initial_memory={"m0": mem}, initial_gpu={"m0": gpu},
                    initial_ssd="all")
    finally:
        S.compose_schedule = real
    outs = [{"nodes": e.payload["nodes"], "classes": {str(x): c for x, c in e.payload["classes"].items()},
             "sources": e.payload["sources"]} for e in res.events if e.kind == "scale_out"]
    return {"label": label, "node_count": n, "initial_gpu": gpu, "initial_memory": mem, "k": k, "b": b,
            "scale_outs": outs[:1], "compose": calls[:1]}


def main():
    doc = {"generator": "tests/golden/make_tiers_golden.py (reference simengine.run, lambda_scale)",
           "cases": [run_case(*c) for c in CASES]}
    with open(os.path.join(HERE, "tiers.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    for c in doc["cases"]:
        so = c["scale_outs"][0] if c["scale_outs"] else None
        print(c["label"], so and so["classes"], so and so["sources"],
              c["compose"][0]["groups"] if c["compose"] else None)


if __name__ == "__main__":
    main()
