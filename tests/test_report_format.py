"""Result files in the reference's layout (cli.py:218-281, §8(f) row 2).

``tests/golden/report/`` holds the reference simulator's own output
(``tests/golden/make_report_golden.py``: ``simengine.run`` +
``cli.write_result``).  Parsing its ``events.log`` with this package and
writing it back with :func:`workload.write_result` must reproduce every file
byte for byte — so a real run's events, written by the same function, are
re-aggregated by the reference's ``blockcast report`` exactly like a
simulated run."""
from pathlib import Path

from paper_2502_09922_b200 import workload as W

GOLD = Path(__file__).parent / "golden" / "report"


def _ref():
    (d,) = [p for p in GOLD.iterdir() if p.is_dir()]
    return d


def test_event_log_round_trip():
    lines = (_ref() / "events.log").read_text().splitlines()
    events = [W.parse_event_line(ln) for ln in lines]
    assert W.event_lines(events) == lines


def test_write_result_matches_reference_files(tmp_path):
    d = _ref()
    events = [W.parse_event_line(ln) for ln in (d / "events.log").read_text().splitlines()]
    end = float([ln for ln in (d / "summary.txt").read_text().splitlines() if ln.startswith("end_s:")][0]
                .split(": ")[1])
    W.write_result(tmp_path, d.name, events, horizon_s=end)
    for name in ("events.log", "summary.txt", "throughput.csv", "allocation.csv"):
        assert (tmp_path / d.name / name).read_bytes() == (d / name).read_bytes(), name
    # per-request rows: the reference writes them from full-precision request
    # state, a log-derived row from 9-decimal event times (cli.py:237) —
    # identical ids, order and blanks, values equal to 1e-8
    ours = (tmp_path / d.name / "metrics_requests.csv").read_text().splitlines()
    ref = (d / "metrics_requests.csv").read_text().splitlines()
    assert ours[0] == ref[0] and len(ours) == len(ref)
    for a, b in zip(ours[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[0] == fb[0]
        for x, y in zip(fa[1:], fb[1:]):
            assert (x == "") == (y == "") and (x == "" or abs(float(x) - float(y)) < 1e-8), (a, b)


def test_request_rows_and_allocation_from_events():
    events = [W.SimEvent(0.0, "allocation", {"allocated_gpus": 2}),
              W.SimEvent(0.01, "request_arrival", {"request": "b", "model": "m"}),
              W.SimEvent(0.01, "request_arrival", {"request": "a", "model": "m"}),
              W.SimEvent(0.05, "token_emitted", {"request": "a", "node": 1, "cold_capacity": True}),
              W.SimEvent(0.07, "token_emitted", {"request": "a", "node": 1, "cold_capacity": True}),
              W.SimEvent(0.07, "request_done", {"request": "a", "node": 1})]
    rows = W.request_rows(events)
    assert [r[0] for r in rows] == ["a", "b"]
    assert abs(rows[0][2] - 0.04) < 1e-12 and rows[0][3] == 0.07
    assert rows[1][2] is None and rows[1][3] is None
    assert W.allocation_samples(events) == [(0.0, 0), (0.0, 2)]


def test_plan_files_match_reference_plan(tmp_path):
    """tools/plan_measure.py writes the reference's `plan` files
    (cli.py:288-339): schedule.txt / pipelines.txt must equal the
    reference's lines for the same (n, k, b) (golden grid, dumped from the
    reference), with the measured lines only appended to summary.txt."""
    import json
    import sys
    sys.path.insert(0, str(Path(__file__).parent.parent / "tools"))
    import plan_measure as PM

    from paper_2502_09922_b200 import scaleout as SO
    grid = {(g["n"], g["k"], g["b"]): g for g in
            json.loads((Path(__file__).parent / "golden" / "schedules.json").read_text())["grid"]}
    for n, k, b in ((8, 1, 16), (8, 2, 16), (4, 1, 4)):
        plan = SO.plan_scale_out("llama3-8b" if b == 16 else "tiny", n, k, b)
        fake = {"plan": plan, "transfer_s": 0.02, "completion_s": {r: 0.02 for r in plan.receivers},
                "first_activation_s": 0.01, "nvlink_frac": 0.8}
        out = tmp_path / f"{n}_{k}_{b}"
        lines = PM.write_plan(out, "m", k, fake)
        g = grid[(n, k, b)]
        assert (out / "schedule.txt").read_text().splitlines() == g["schedule_lines"]
        assert (out / "pipelines.txt").read_text().splitlines() == g["pipeline_lines"]
        assert f"step_count: {g['summary']['step_count']}" in lines
        assert any(ln.startswith("measured_transfer_s:") for ln in lines)
