"""GPU: the reference simulator with the B200 hot path plugged in
(SURVEY.md 8(f) row 1). integration/des_gpu_main.cpp runs the reference's own
config/trace/arrival/DES/CSV code with every query scored by K4 in one launch
and every control tick planned by K1 through ds_b200::GpuPlannerPolicy. The
CSVs must be byte-identical to the stock reference run (digests from
tests/golden/des_inputs.npz, = SURVEY Appendix A.1)."""
import hashlib
import os
import subprocess

import numpy as np
import pytest

from oracle import des_inputs, lib

pytestmark = pytest.mark.gpu

EXE = os.path.join(lib.HERE, "_ref", "des_gpu")
needs_exe = pytest.mark.skipif(not os.path.exists(EXE),
                               reason="oracle/_ref/des_gpu not built (needs /root/reference)")


def md5(path):
    return hashlib.md5(open(path, "rb").read()).hexdigest()


@pytest.fixture(scope="module")
def inputs(tmp_path_factory, golden):
    root = str(tmp_path_factory.mktemp("des"))
    g = golden("des_inputs")
    return root, des_inputs.write_inputs(root, g), g


@needs_exe
@pytest.mark.parametrize("name", ["cascade1", "cascade2", "cascade3"])
def test_drop_in_des_csvs_byte_identical(inputs, name):
    root, cfgs, g = inputs
    out = os.path.join(root, "gpu_" + name)
    r = subprocess.run([EXE, "--config", cfgs[name], "--out", out, "--mode", "gpu"], cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    print(r.stdout.strip())
    for csv in ("intervals", "plans", "queries"):
        assert md5(os.path.join(out, csv + ".csv")) == str(g[f"md5_{name}_{csv}"]), csv


@needs_exe
@pytest.mark.parametrize("policy", ["diffserve_static", "clipper_light", "clipper_heavy",
                                    "proteus_like", "abl_static_threshold",
                                    "abl_aimd_batching", "abl_no_queuing_model"])
def test_every_policy_kind_matches_stock_reference(inputs, policy):
    """GpuPlannerPolicy vs the reference's own make_policy() on the same box."""
    root, cfgs, _ = inputs
    outs = {}
    for mode in ("cpu", "gpu"):
        out = os.path.join(root, f"{mode}_{policy}")
        r = subprocess.run([EXE, "--config", cfgs["cascade1"], "--out", out, "--mode", mode,
                            "--policy", policy, "--seed", "3"], cwd=root, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs[mode] = out
    for csv in ("intervals", "plans", "queries"):
        assert md5(os.path.join(outs["cpu"], csv + ".csv")) == \
            md5(os.path.join(outs["gpu"], csv + ".csv")), csv
