"""Golden result files from the reference's own writer (run HERE only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_report_golden.py

Runs the reference simulator (``blockcast.simengine.run``) on a small
λScale burst and writes its output with ``blockcast.cli.write_result`` into
``tests/golden/report/`` — the fixture ``tests/test_report_format.py``
compares this package's writer against, byte for byte.
"""
import os
import shutil
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from blockcast import cli, simengine as S, workload as W  # noqa: E402
from blockcast.multicast import ModelSpec  # noqa: E402

out = Path(os.path.dirname(os.path.abspath(__file__))) / "report"
shutil.rmtree(out, ignore_errors=True)
cluster = S.ClusterSpec(node_count=8)
model = ModelSpec("llama3-8b", 16_060_522_496, 32)
trace = W.synth_burst(0.5, 20.0, [1.0], 6.0, seed=7, model_ids=("llama3-8b",), spike_duration_s=1.0,
                      output_tokens=(4, 8))
res = S.run(cluster, [model], "lambda_scale", trace, S.AutoscalePolicy(), seed=3, k=2,
            initial_gpu={"llama3-8b": [0]})
cli.write_result(out, res)
print(out, len(res.events), "events,", len(res.request_rows), "requests")
