"""TEST INFRASTRUCTURE ONLY -- writes the reference's experiment inputs
(profile file, three cascade configs, demand traces) into a directory, from
values committed in tests/golden/des_inputs.npz, so the drop-in DES run
(oracle/_ref/des_gpu, integration/) can be replayed on a box without
/root/reference. The writer's output parses to the same doubles as the
reference's own files (proj/configs/*, proj/traces/*); oracle/make_golden.py
checks that by running the reference on both and comparing CSV digests."""
from __future__ import annotations

import os

import numpy as np

CFG_KEYS = ["profiles", "cascade", "trace", "policy", "servers", "seed", "out_dir",
            "arrival_mode", "control_interval_seconds", "ewma_alpha", "overprovision_lambda",
            "threshold_grid_step", "deferral_decay", "bill_formed_batch",
            "confidence_fidelity", "noise_sigma"]


def write_inputs(root: str, g: dict) -> dict:
    """Writes configs/ and traces/ under root; returns {cascade: cfg path}."""
    os.makedirs(os.path.join(root, "configs"), exist_ok=True)
    os.makedirs(os.path.join(root, "traces"), exist_ok=True)
    prof = []
    for name in ("cascade1", "cascade2", "cascade3"):
        lt = g[f"{name}_light"]
        ht = g[f"{name}_heavy"]
        prof += ["cascade {", f"  name = {name}", f"  slo_seconds = {float(g[name + '_slo'])!r}",
                 "  light.latency = { " + ", ".join(f"{int(b)}: {float(e)!r}" for b, e in lt) + " }",
                 "  heavy.latency = { " + ", ".join(f"{int(b)}: {float(e)!r}" for b, e in ht) + " }",
                 "  deferral.samples = [ " + ", ".join(repr(float(x)) for x in g["prior"]) + " ]",
                 "}", ""]
    with open(os.path.join(root, "configs", "cascades.profiles"), "w") as f:
        f.write("\n".join(prof))
    for tname in ("trace_4to32qps", "trace_1to8qps", "trace_8to24qps"):
        with open(os.path.join(root, "traces", tname + ".txt"), "w") as f:
            f.write("\n".join(repr(float(x)) for x in g[tname]) + "\n")
    cfgs = {}
    for name, trace in (("cascade1", "trace_4to32qps"), ("cascade2", "trace_4to32qps"),
                        ("cascade3", "trace_1to8qps")):
        vals = dict(profiles="configs/cascades.profiles", cascade=name,
                    trace=f"traces/{trace}.txt", policy="diffserve", servers="16", seed="1",
                    out_dir=f"out/{name}", arrival_mode="poisson",
                    control_interval_seconds="10", ewma_alpha="0.5",
                    overprovision_lambda="1.05", threshold_grid_step="0.01",
                    deferral_decay="0.999", bill_formed_batch="true",
                    confidence_fidelity="0.35", noise_sigma="0.12")
        path = os.path.join(root, "configs", f"{name}.cfg")
        with open(path, "w") as f:
            f.write("\n".join(f"{k} = {vals[k]}" for k in CFG_KEYS) + "\n")
        cfgs[name] = path
    return cfgs
