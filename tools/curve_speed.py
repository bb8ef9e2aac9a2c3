"""Times ds_curve_observe_device (K3) on 1M latent confidences at decay 0.999
and checks the curve bit for bit against the C restatement."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lib  # noqa: E402
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    ctx = native.Context(0)
    L = native.lib()
    conf = ctx.score_latent(workloads.query_model(), 0, n)
    prior = workloads.uniform_prior()
    want = prior.copy()
    lib.port().dso_curve_observe(abi.ptr(want), abi.ptr(conf), n, 0.999)
    dconf = torch.from_numpy(conf).cuda()
    p_t = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
    c_t = torch.empty_like(p_t)
    st = torch.cuda.ExternalStream(ctx.stream)

    def run():
        with torch.cuda.stream(st):
            c_t.copy_(p_t)
            native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(c_t.data_ptr()),
                                                   native.c_p(dconf.data_ptr()), abi.CONF_F64, n,
                                                   0.999, native.c_p(ctx.stream)))
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        run()
    b.record(st)
    torch.cuda.synchronize()
    got = c_t.cpu().numpy().view(abi.CURVE)[0]
    ok = got.tobytes() == want.tobytes()
    print(f"{os.environ.get('DS_EXTRA_NVCC', 'default')}: curve replay {n} obs: "
          f"{a.elapsed_time(b) / 3:.3f} ms, bit-exact vs port: {ok}")


if __name__ == "__main__":
    main()
