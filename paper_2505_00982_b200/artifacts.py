"""Run artifacts and their reports, in the reference's schemas.

harness.cpp:316-440 writes four files per run: ``metrics.csv`` (one MetricsRow per inner epoch),
``ledger.csv`` (CommLedger rows), ``memory.csv`` (SlotMeter peaks per rank) and ``summary.json``;
``memory_report`` / ``comm_report`` (harness.cpp:494-593) validate them. The writers here produce
the same headers, cell formats (``%.17g``, empty cell for NaN / negative outer/inner) and summary
keys from a device run, so the reference's reports read GPU runs unchanged. Two differences are
inherent to the device decomposition and are spelled out where they matter:

* memory is accounted per GPU rank (the basis is sharded over G GPUs, not over the C logical
  workers), so ``memory_report`` bounds D_shard by ceil(n / G) (m + 1);
* the ledger records the NCCL rounds the device path issues: all_gather(v_i),
  reduce_scatter(Hv), all-reduces of the (m + 2)-float GS partials and of beta^2 per pass, and per
  step reduce_scatter(g) / all-reduces of r floats / all_gather(w_a). A single GPU communicates
  nothing, so its ledger is empty.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

from .api import (Context, Dataset, TrainerConfig, TrainingDiverged, TrainResult, Trainer, lanczos_budget,
                  shard_for_rank)


def format_double(x: float) -> str:
    """harness.cpp:19-23 (``%.17g``)."""
    return "%.17g" % x


def _metric_cell(x: float) -> str:
    return "" if math.isnan(x) else format_double(x)


@dataclass
class RunPaths:
    """harness.cpp:316-318."""
    metrics_csv: str
    ledger_csv: str
    memory_csv: str
    summary_json: str

    @staticmethod
    def in_dir(d: str) -> "RunPaths":
        return RunPaths(os.path.join(d, "metrics.csv"), os.path.join(d, "ledger.csv"),
                        os.path.join(d, "memory.csv"), os.path.join(d, "summary.json"))


def write_metrics_csv(path: str, trainer: str, res: TrainResult) -> None:
    """harness.cpp:324-340."""
    with open(path, "w") as f:
        f.write("trainer,outer_k,inner_l,epoch,train_loss,train_acc,residual_norm,wallclock_ms,ese_refresh_flag\n")
        for i in range(len(res.loss)):
            ok = int(res.outer_k[i]) if res.outer_k is not None else -1
            il = int(res.inner_l[i]) if res.inner_l is not None else -1
            wall = float(res.wallclock_ms[i]) if res.wallclock_ms is not None else 0.0
            f.write(f"{trainer},{ok if ok >= 0 else ''},{il if il >= 0 else ''},{int(res.epoch[i])},"
                    f"{format_double(float(res.loss[i]))},{_metric_cell(float(res.acc[i]))},"
                    f"{_metric_cell(float(res.residual_norm[i]))},{format_double(wall)},"
                    f"{1 if res.ese_refresh[i] else 0}\n")


def write_ledger_csv(path: str, rows: Sequence[tuple]) -> None:
    """harness.cpp:342-350; rows are (event, op, floats, rank, sent, received)."""
    with open(path, "w") as f:
        f.write("event_index,op,floats,rank,sent,received\n")
        for r in rows:
            f.write(",".join(str(x) for x in r) + "\n")


def write_memory_csv(path: str, meters: Sequence[Dict[str, int]]) -> None:
    """harness.cpp:352-361 (objects in std::map order)."""
    with open(path, "w") as f:
        f.write("rank,object,peak_slots\n")
        for r, meter in enumerate(meters):
            for name in sorted(meter):
                f.write(f"{r},{name},{meter[name]}\n")


def summary_dict(cfg: TrainerConfig, *, trainer: str, workers: int, gpus: int, seed: int, schedule: str,
                 problem_kind: str, n: int, samples: int, loss_target: float) -> dict:
    """The pre-run keys of run_experiment (harness.cpp:376-389)."""
    m = 0
    if cfg.k + cfg.l > 0:
        m = cfg.lanczos_m if cfg.lanczos_m else lanczos_budget(cfg.k, cfg.l, n)
    b0, e0 = shard_for_rank(samples, workers, 0)
    return {"trainer": trainer, "workers": workers, "gpus": gpus, "seed": seed, "schedule": schedule,
            "problem_kind": problem_kind, "n": n, "samples": samples, "k": cfg.k, "l": cfg.l, "lanczos_m": m,
            "rounds_per_epoch": (e0 - b0 + cfg.batch_size - 1) // cfg.batch_size, "loss_target": loss_target}


def finish_summary(summary: dict, res: TrainResult, meters: Sequence[Dict[str, int]], loss_target: float) -> dict:
    """The post-run keys (harness.cpp:407-436)."""
    summary["aborted"] = False
    summary["epochs_run"] = len(res.loss)
    summary["ese_refreshes"] = res.ese_refreshes
    summary["gs_flops"] = res.gs_flops
    summary["safeguard_passes"] = res.safeguard_passes
    summary["final_loss"] = res.final_loss()
    summary["final_accuracy"] = res.final_accuracy()
    e = res.epochs_to_loss(loss_target)
    summary["epochs_to_target"] = e
    summary["modeled_ms_at_target"] = float(res.wallclock_ms[e - 1]) if e is not None else None
    summary["modeled_total_ms"] = float(res.wallclock_ms[-1]) if len(res.loss) else 0.0
    summary["raw_wallclock_ms"] = res.raw_wallclock_ms
    summary["d_shard_slots_per_rank"] = [int(mt.get("D_shard", 0)) for mt in meters]
    return summary


def _dump(path: str, obj: dict) -> None:
    with open(path, "w") as f:  # nlohmann::json objects are key-sorted; dump(2)
        f.write(json.dumps(obj, indent=2, sort_keys=True) + "\n")


def run_experiment(ctx: Context, cfg: TrainerConfig, oracle, data: Dataset, w0, out_dir: str, *, workers: int = 1,
                   seed: Optional[int] = None, problem_kind: str = "mlp", loss_target: float = 0.0,
                   schedule: str = "nccl") -> int:
    """run_experiment (harness.cpp:364-440) on the device path: train, then write the four artifacts.
    Returns 0, or 2 with an ``aborted`` summary when training diverges (harness.cpp:396-402)."""
    import time
    os.makedirs(out_dir, exist_ok=True)
    paths = RunPaths.in_dir(out_dir)
    n = oracle.dim()
    summary = summary_dict(cfg, trainer=cfg.kind, workers=workers, gpus=ctx.world, seed=cfg.seed if seed is None
                           else seed, schedule=schedule, problem_kind=problem_kind, n=n, samples=data.size(),
                           loss_target=loss_target)
    ctx.reset_accounting()
    tr = Trainer(ctx, cfg, oracle, data, w0, workers)
    try:
        t0 = time.perf_counter()
        try:
            tr.run()
        except TrainingDiverged as e:
            summary["aborted"] = True
            summary["abort_reason"] = str(e)
            _dump(paths.summary_json, summary)
            return 2
        res = tr.result()
        res.raw_wallclock_ms = (time.perf_counter() - t0) * 1e3
    finally:
        tr.close()
    meters = [ctx.memory()]
    if ctx.world > 1:  # every rank's D_shard peak, in rank order (the reference lists one per worker)
        slots = ctx.allgather_host([float(meters[0].get("D_shard", 0))])[:, 0]
        meters = [dict(meters[0]) if r == ctx.rank else {"D_shard": int(v)} for r, v in enumerate(slots)]
    write_metrics_csv(paths.metrics_csv, cfg.kind, res)
    write_ledger_csv(paths.ledger_csv, ctx.ledger())
    write_memory_csv(paths.memory_csv, meters)
    _dump(paths.summary_json, finish_summary(summary, res, meters, loss_target))
    return 0


# ------------------------------------------------------------------------------ reports
def memory_report(run_dirs: Sequence[str]) -> str:
    """memory_report (harness.cpp:494-524): the measured D_shard peak must equal ceil(n / G) (m + 1)
    and must not grow as G grows across the given runs (G = the GPU count of each run)."""
    lines = ["C  n      m   D_shard_slots  bound=ceil(n/C)*(m+1)  status"]
    prev, all_ok = -1, True
    for d in run_dirs:
        with open(RunPaths.in_dir(d).summary_json) as f:
            s = json.load(f)
        n, m = int(s["n"]), int(s["lanczos_m"])
        g = int(s.get("gpus", s["workers"]))
        slots = s.get("d_shard_slots_per_rank", [])
        measured = max(slots) if slots else 0
        bound = ((n + g - 1) // g) * (m + 1)
        ok = measured == bound and (prev < 0 or measured <= prev)
        all_ok = all_ok and ok
        prev = measured
        lines.append("%-2d %-6d %-3d %-14d %-22d %s" % (g, n, m, measured, bound, "OK" if ok else "MISMATCH"))
    lines.append("memory accounting: OK" if all_ok else "memory accounting: MISMATCH")
    return "\n".join(lines) + "\n"


def load_ledger(path: str) -> List[tuple]:
    rows = []
    with open(path) as f:
        next(f)
        for line in f:
            line = line.strip()
            if not line:
                continue
            ev, op, fl, rk, se, rc = line.split(",")
            rows.append((int(ev), op, int(fl), int(rk), int(se), int(rc)))
    return rows


def comm_report(run_dir: str, reorth_safeguard: bool = True, mlp_operator: bool = True) -> str:
    """comm_report (harness.cpp:526-591) for the device decomposition (module docstring).

    Expected rounds at G > 1 (every rank records each round once): per refresh one all_reduce(1) for
    ||v_1||^2, m all_gather(v_i), m reduce_scatter(Hv) (MLP operator), per GS pass (1, or 2 with the
    safeguard: its second pass is a predicated launch, so its collectives always run) m all_reduce of
    the GS partials and m all_reduce(beta^2), and one all_gather of the sign-argmax pairs. At G = 1
    every count is zero. Traffic must be conserved (sent == received)."""
    paths = RunPaths.in_dir(run_dir)
    with open(paths.summary_json) as f:
        s = json.load(f)
    rows = load_ledger(paths.ledger_csv)
    g = int(s.get("gpus", 1))
    refreshes, m = int(s["ese_refreshes"]), int(s["lanczos_m"])
    passes = 2 if reorth_safeguard else 1
    ops: Dict[str, int] = {}
    by_floats: Dict[tuple, int] = {}
    sent = sum(r[4] for r in rows)
    received = sum(r[5] for r in rows)
    for r in rows:
        ops[r[1]] = ops.get(r[1], 0) + 1
        by_floats[(r[1], r[2])] = by_floats.get((r[1], r[2]), 0) + 1
    n = int(s["n"])
    stride = 2 * (m + 2)  # GS partial row: [r_0..r_i, ||h||^2] and the Gram column (lanczos.cu)
    scale = 1 if g > 1 else 0
    n_pad = (n + g - 1) // g * g
    # all_gather(v_i) and all_gather(w_a) both move n_pad floats: the v_i share is refreshes * m
    checks = [
        ("all_gather(n)", by_floats.get(("all_gather", n_pad), 0), None),
        ("reduce(GS)", by_floats.get(("all_reduce", stride), 0), refreshes * m * passes * scale),
        ("reduce(beta)", by_floats.get(("all_reduce", 1), 0), (refreshes * m * passes + refreshes) * scale),
    ]
    if mlp_operator:
        checks.append(("reduce_scat(n)", by_floats.get(("reduce_scatter", n_pad), 0), None))
    out = ["op             events  expected"]
    ok = True
    for name, got, want in checks:
        if want is None:
            out.append("%-14s %-7d %-8s %s" % (name, got, ">= %d" % (refreshes * m * scale), "info"))
            continue
        good = got == want
        ok = ok and good
        out.append("%-14s %-7d %-8d %s" % (name, got, want, "OK" if good else "MISMATCH"))
    for op in sorted(ops):
        out.append("%-14s %-7d %-8s %s" % (op, ops[op], "-", "total"))
    out.append("floats sent %d, received %d%s" % (sent, received, " (conserved)" if sent == received
                                                   else " (NOT conserved)"))
    ok = ok and sent == received
    out.append("communication ledger: OK" if ok else "communication ledger: MISMATCH")
    return "\n".join(out) + "\n"
