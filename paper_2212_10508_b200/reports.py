"""Parareal run reports in the reference's file formats (host side).

The reference writes, per parareal run (cli.py:888-930): ``trajectory.csv``
(model.py:158-176, here ``model.write_trajectory_csv``), ``history.csv``
(``_write_history_csv``, cli.py:784-790: slab, iteration, delta with 17
significant digits) and ``result.json`` (``_write_json`` / ``_jsonable`` /
``_slab_payload`` / ``_state_payload``, cli.py:761-807: sorted keys, indent 2,
numpy scalars and arrays as plain JSON numbers and lists).  The node states
come off the device once, at the end of the run (``PararealResult.trajectory``).
"""

from __future__ import annotations

import csv
import json
from pathlib import Path
from typing import Any

import numpy as np

from .accounting import adaptive_gain, classic_gain
from .model import write_trajectory_csv


def _plain(obj: Any) -> Any:
    if isinstance(obj, dict):
        return {str(k): _plain(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_plain(v) for v in obj]
    if isinstance(obj, np.ndarray):
        return [_plain(v) for v in obj.tolist()]
    if isinstance(obj, np.floating):
        return float(obj)
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, Path):
        return str(obj)
    return obj


def write_json(path, payload: dict) -> Path:
    path = Path(path)
    path.write_text(json.dumps(_plain(payload), indent=2, sort_keys=True) + "\n")
    return path


def write_history_csv(path, history) -> Path:
    path = Path(path)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(("slab", "iteration", "delta"))
        for slab, iteration, delta in history:
            w.writerow((str(slab), str(iteration), format(delta, ".17g")))
    return path


def slab_payload(result) -> list:
    return [{"slab_index": s.slab_index, "n_init": s.n_init, "n_final": s.n_final, "k_conv": s.k_conv,
             "attempts": [[a.n_final, a.iterations] for a in s.attempts]} for s in result.slabs]


def state_payload(state) -> dict:
    return {"q": state.q, "p": state.p}


def parareal_payload(result, experiment: str, n_windows: int, window_dt: float, delta_conv: float,
                     delta_expl, cost_fine: float, cost_coarse: float) -> dict:
    """The ``result.json`` payload of a parareal run (cli.py:907-928)."""
    gain = None
    if result.converged:
        if experiment == "parareal_adaptive":
            gain = adaptive_gain(result.slabs, n_windows, cost_fine, cost_coarse)
        else:
            gain = classic_gain(n_windows, result.slabs[0].k_conv, cost_fine, cost_coarse)
    return {
        "experiment": experiment,
        "n_windows": n_windows,
        "window_dt": window_dt,
        "delta_conv": delta_conv,
        "delta_expl": delta_expl,
        "converged": result.converged,
        "n_slab": result.n_slab,
        "total_iterations": result.total_iterations,
        "slabs": slab_payload(result),
        "gain": None if gain is None else gain.as_dict(),
        "final": state_payload(result.trajectory[n_windows]),
    }


def write_parareal_report(out_dir, result, experiment: str, params, config, pair) -> list:
    """trajectory.csv, history.csv and result.json of one run; returns the paths."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    traj = out / "trajectory.csv"
    write_trajectory_csv(result.trajectory, traj, params.window_dt)
    hist = write_history_csv(out / "history.csv", result.error_history)
    payload = parareal_payload(result, experiment, config.n_windows, params.window_dt, config.delta_conv,
                               config.delta_expl, pair.cost_fine, pair.cost_coarse)
    return [traj, hist, write_json(out / "result.json", payload)]
