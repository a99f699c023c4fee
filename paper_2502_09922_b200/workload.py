"""Request traces and serving metrics — the hot-path subset of
``blockcast.workload`` (pkg/src/blockcast/workload.py).

The real serving runtime (:mod:`.serving`) emits :class:`SimEvent` records
with wall-clock timestamps in exactly the reference's shape
(``request_arrival``, ``token_emitted{request,node,cold_capacity}``,
``request_done``, ``mode_switch``, ``transfer_step_done``, ``allocation``), so
:func:`aggregate` computes TTFT percentiles (nearest rank), the 100 ms
tokens/s timeline, ramp time and GPU-seconds with the reference definitions
(workload.py:165-233).  :func:`synth_burst` reproduces the reference's seeded
thinned-Poisson trace draw for draw (workload.py:122-162).
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

from .errors import IncompleteLogError, InvalidArgumentError

THROUGHPUT_WINDOW_S = 0.1


@dataclass(frozen=True)
class TraceRecord:
    request_id: str
    arrival_s: float
    model_id: str
    prompt_tokens: int
    output_tokens: int


@dataclass(frozen=True)
class SimEvent:
    time_s: float
    kind: str
    payload: dict


@dataclass
class MetricsReport:
    label: str
    requests_arrived: int = 0
    requests_completed: int = 0
    requests_in_flight: int = 0
    total_tokens: int = 0
    ttft_samples: list = field(default_factory=list)
    ttft_p50: float | None = None
    ttft_p90: float | None = None
    ttft_p99: float | None = None
    throughput_timeline: list = field(default_factory=list)
    gpu_seconds_cumulative: float = 0.0
    first_token_s: float | None = None
    ramp_first_serve_s: float | None = None
    end_s: float = 0.0


def nearest_rank(samples: list, percentile: float):
    """The ceil(p/100 * n)-th smallest sample (workload.py:53-61)."""
    if not samples:
        return None
    if not (0 < percentile <= 100):
        raise InvalidArgumentError("percentile must be in (0, 100]")
    ranked = sorted(samples)
    return ranked[math.ceil(percentile / 100.0 * len(ranked)) - 1]


def synth_burst(base_rps: float, spike_rps: float, spike_times: list, duration_s: float,
                seed: int, *, spike_duration_s: float = 60.0, model_ids: tuple = ("m0",),
                prompt_tokens: tuple = (128, 128),
                output_tokens: tuple = (32, 32)) -> list:
    """Seeded base-rate + rectangular-spike arrivals by Poisson thinning."""
    if duration_s <= 0:
        raise InvalidArgumentError("duration_s must be positive")
    if base_rps < 0 or spike_rps < 0:
        raise InvalidArgumentError("rates must be non-negative")
    ceiling = base_rps + (spike_rps if spike_times else 0.0)
    if ceiling <= 0:
        return []

    def rate_at(t):
        return base_rps + spike_rps * sum(1 for s0 in spike_times
                                          if s0 <= t < s0 + spike_duration_s)

    draw = random.Random(seed)
    trace = []
    t = 0.0
    while True:
        t += draw.expovariate(ceiling)
        if t >= duration_s:
            return trace
        if draw.random() * ceiling <= rate_at(t):
            n = len(trace)
            trace.append(TraceRecord(f"r{n}", t, model_ids[n % len(model_ids)],
                                     draw.randint(*prompt_tokens), draw.randint(*output_tokens)))


def integrate_allocation(samples: list, end_s: float) -> float:
    """Step integral of (time, allocated devices) change points up to ``end_s``."""
    area = 0.0
    for (t0, v), (t1, _) in zip(samples, samples[1:]):
        area += v * (t1 - t0)
    if samples:
        t_last, v_last = samples[-1]
        area += v_last * max(0.0, end_s - t_last)
    return area


def aggregate(events: list, label: str = "run", horizon_s: float | None = None) -> MetricsReport:
    """Fold an event stream into TTFT / throughput / GPU-seconds (workload.py:165-222)."""
    rep = MetricsReport(label)
    arrived: dict = {}
    first: dict = {}
    finished: set = set()
    stamps: list = []
    alloc: list = []
    end = 0.0 if horizon_s is None else horizon_s
    for ev in events:
        end = max(end, ev.time_s)
        kind = ev.kind
        if kind == "request_arrival":
            arrived[ev.payload["request"]] = ev.time_s
        elif kind == "token_emitted":
            rid = ev.payload["request"]
            stamps.append(ev.time_s)
            if rid not in first:
                first[rid] = ev.time_s
                if rep.first_token_s is None:
                    rep.first_token_s = ev.time_s
                if ev.payload.get("cold_capacity") and rep.ramp_first_serve_s is None:
                    rep.ramp_first_serve_s = ev.time_s
        elif kind == "request_done":
            finished.add(ev.payload["request"])
        elif kind == "allocation":
            alloc.append((ev.time_s, ev.payload["allocated_gpus"]))
    open_reqs = set(arrived) - finished
    if open_reqs and horizon_s is None:
        raise IncompleteLogError(
            f"{len(open_reqs)} request(s) have no terminal event and no horizon was given")
    rep.requests_arrived = len(arrived)
    rep.requests_completed = len(finished)
    rep.requests_in_flight = len(open_reqs)
    rep.total_tokens = len(stamps)
    rep.ttft_samples = sorted(first[r] - arrived[r] for r in first if r in arrived)
    rep.ttft_p50 = nearest_rank(rep.ttft_samples, 50)
    rep.ttft_p90 = nearest_rank(rep.ttft_samples, 90)
    rep.ttft_p99 = nearest_rank(rep.ttft_samples, 99)
    rep.end_s = end
    stamps.sort()
    nwin = int(math.ceil(end / THROUGHPUT_WINDOW_S)) if end > 0 else 0
    cursor = 0
    for w in range(nwin):
        edge = (w + 1) * THROUGHPUT_WINDOW_S
        start = cursor
        while cursor < len(stamps) and stamps[cursor] <= edge:
            cursor += 1
        rep.throughput_timeline.append((edge, (cursor - start) / THROUGHPUT_WINDOW_S))
    rep.gpu_seconds_cumulative = integrate_allocation(alloc, end)
    return rep


# ---------------------------------------------------------------------------
# Result files in the reference's layout (cli.py:218-281), so the reference's
# ``blockcast report <outdir>`` (cli.py:413-432) re-aggregates a REAL run the
# same way it aggregates a simulated one.

def fmt(x) -> str:
    """cli.py:218-223 number formatting."""
    if x is None:
        return ""
    if isinstance(x, float):
        return f"{x:.9g}"
    return str(x)


def event_lines(events: list) -> list:
    """``events.log`` lines: ``time,kind,k=json;k=json`` (cli.py:231-238)."""
    import json
    out = []
    for e in events:
        payload = ";".join(f"{k}={json.dumps(v, sort_keys=True, separators=(',', ':'))}"
                           for k, v in sorted(e.payload.items()))
        out.append(f"{e.time_s:.9f},{e.kind},{payload}")
    return out


def parse_event_line(line: str) -> SimEvent:
    """Inverse of :func:`event_lines` (cli.py:241-248)."""
    import json
    t, kind, payload = line.split(",", 2)
    d = {}
    if payload:
        for item in payload.split(";"):
            k, v = item.split("=", 1)
            d[k] = json.loads(v)
    return SimEvent(float(t), kind, d)


def summary_block(r: MetricsReport) -> list:
    """``summary.txt`` lines (cli.py:251-265)."""
    return [
        f"strategy: {r.label}",
        f"requests_arrived: {r.requests_arrived}",
        f"requests_completed: {r.requests_completed}",
        f"requests_in_flight: {r.requests_in_flight}",
        f"total_tokens: {r.total_tokens}",
        f"ttft_p50_s: {fmt(r.ttft_p50)}",
        f"ttft_p90_s: {fmt(r.ttft_p90)}",
        f"ttft_p99_s: {fmt(r.ttft_p99)}",
        f"first_token_s: {fmt(r.first_token_s)}",
        f"time_to_first_served_s: {fmt(r.ramp_first_serve_s)}",
        f"gpu_seconds_total: {fmt(r.gpu_seconds_cumulative)}",
        f"end_s: {fmt(r.end_s)}",
    ]


def request_rows(events: list) -> list:
    """(request_id, arrival_s, ttft_s, completion_s) per request in (arrival,
    id) order — the reference builds them from its request table
    (simengine.py:765-769); a real run derives the same from its events."""
    arrival, first, done = {}, {}, {}
    for e in events:
        rid = e.payload.get("request")
        if e.kind == "request_arrival":
            arrival[rid] = e.time_s
        elif e.kind == "token_emitted" and rid not in first:
            first[rid] = e.time_s
        elif e.kind == "request_done":
            done[rid] = e.time_s
    return [(rid, arrival[rid], None if rid not in first else first[rid] - arrival[rid], done.get(rid))
            for rid in sorted(arrival, key=lambda r: (arrival[r], r))]


def allocation_samples(events: list) -> list:
    """(time, allocated GPUs) change points: (0, 0) then every ``allocation``
    event (simengine.py:284, 295-298)."""
    return [(0.0, 0)] + [(e.time_s, e.payload["allocated_gpus"]) for e in events if e.kind == "allocation"]


def write_result(outdir, label: str, events: list, report: MetricsReport | None = None,
                 horizon_s: float | None = None) -> None:
    """Write ``<outdir>/<label>/{metrics_requests.csv, throughput.csv,
    allocation.csv, events.log, summary.txt}`` exactly as cli.write_result
    (cli.py:268-281) does for a simulated run."""
    from pathlib import Path
    d = Path(outdir) / label
    d.mkdir(parents=True, exist_ok=True)
    if report is None:
        report = aggregate(events, label=label, horizon_s=horizon_s)

    def write(name, lines):
        (d / name).write_text("\n".join(lines) + ("\n" if lines else ""))

    write("metrics_requests.csv", ["request_id,arrival_s,ttft_s,completion_s"] +
          [f"{rid},{fmt(a)},{fmt(t)},{fmt(c)}" for rid, a, t, c in request_rows(events)])
    write("throughput.csv", ["time_s,tokens_per_s"] +
          [f"{fmt(t)},{fmt(v)}" for t, v in report.throughput_timeline])
    write("allocation.csv", ["time_s,allocated_gpus"] +
          [f"{fmt(t)},{v}" for t, v in allocation_samples(events)])
    write("events.log", event_lines(events))
    write("summary.txt", summary_block(report))
