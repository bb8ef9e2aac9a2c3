"""Per-phase clock64 trace of disc_kernel CTA 0 (debug build path).

Prints, per token tile, the cycle offsets of: A-builder (r1_free seen, first
chunk stored, last chunk stored), epilogue (acc ready / done for E1, E2_0..3,
E3) and the MMA issuer (tile start, GEMM1 issued, epi_done seen / GEMM2 issued
per j, GEMM3 issued)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    ctx = native.Context(0)
    L = native.lib()
    L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                                ctypes.c_int32] + [ctypes.c_void_p] * 3
    disc = native.Discriminator(ctx, 2024)
    img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
    native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512,
                                          native.c_p(img.data_ptr()), native.c_p(ctx.stream)))
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    tr = torch.zeros(8 * 8 * 16 + 5 * 160, dtype=torch.int64, device="cuda")
    for _ in range(2):
        native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr()), n, 512, 512,
                                            native.c_p(conf.data_ptr()), native.c_p(tr.data_ptr()),
                                            native.c_p(ctx.stream)))
    ctx.synchronize()
    tall = tr.cpu().numpy()
    t = tall[:8 * 8 * 16].reshape(8, 8, 16)
    cta = tall[8 * 8 * 16:8 * 8 * 16 + 480].reshape(160, 3)
    base = t[2, 0, 0]
    names = {0: ["c0_start", "c11_stored"],
             1: ["E1_rdy", "E1_done", "E20_rdy", "E20_done", "E21_rdy", "E21_done", "E22_rdy",
                 "E22_done", "E23_rdy", "E23_done", "E3_rdy", "E3_done"],
             2: ["start", "G1_iss", "G33prev_iss", "E1_seen", "dr0", "rd0", "dr1", "rd1", "dr2",
                 "rd2", "dr3"]}
    for tile in range(8):
        print(f"--- tile {tile}")
        for role in (2, 1, 0):
            vals = t[role, tile]
            s = "  ".join(f"{nm}={int(vals[i] - base) if vals[i] else -1}"
                          for i, nm in enumerate(names[role]))
            print(f"  role{role}: {s}")
    print("per-tile cycles (MMA start deltas):", np.diff(t[2, :, 0]).tolist())
    used = cta[:, 0] > 0
    st = cta[used, 0]
    dur = (cta[used, 1] - cta[used, 0]) / 1e3
    print(f"CTAs {used.sum()}: start spread {(st.max() - st.min()) / 1e3:.1f} us; duration us "
          f"min {dur.min():.0f} median {np.median(dur):.0f} max {dur.max():.0f}")
    order = np.argsort(-dur)[:6]
    print("slowest CTAs (bid, smid, us):", [(int(i), int(cta[i, 2]), round(float(dur[i]))) for i in order])
    for tile in (6,):
        print(f"tile {tile} weight stages: producer issue / MMA b_full seen / latency")
        for k in range(16):
            print(f"  s{k:2d}: {int(t[6, tile, k] - base):8d} {int(t[7, tile, k] - base):8d} "
                  f"{int(t[7, tile, k] - t[6, tile, k]):6d}")
    for tile in (6,):
        print(f"tile {tile} per-chunk: a_empty_ok / a_full_arrive / mma_a_full_seen")
        for c in range(12):
            print(f"  c{c:2d}: {int(t[3, tile, c] - base):8d} {int(t[4, tile, c] - base):8d} "
                  f"{int(t[5, tile, c] - base):8d}")


if __name__ == "__main__" and not (len(sys.argv) > 2 and sys.argv[2] == "prologue"):
    main()


def prologue(n=5000):
    """Tile 0 of CTA 0 in detail: the A-builder's first loads / prefetches and
    per-chunk store times, the MMA's per-chunk waits, the weight stages."""
    ctx = native.Context(0)
    L = native.lib()
    L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                                ctypes.c_int32] + [ctypes.c_void_p] * 3
    disc = native.Discriminator(ctx, 2024)
    img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
    native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512,
                                          native.c_p(img.data_ptr()), native.c_p(ctx.stream)))
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    tr = torch.zeros(8 * 8 * 16 + 5 * 160, dtype=torch.int64, device="cuda")
    for _ in range(2):
        native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr()), n, 512, 512,
                                            native.c_p(conf.data_ptr()), native.c_p(tr.data_ptr()),
                                            native.c_p(ctx.stream)))
    ctx.synchronize()
    tall = tr.cpu().numpy()
    t = tall[:8 * 8 * 16].reshape(8, 8, 16)
    c0 = tall[8 * 8 * 16 + 480]   # CTA 0's clock64 at its start
    rel = lambda v: int(v - c0) if v else -1   # noqa: E731
    print("CTA 0 tile 0, cycles after the CTA's first instruction:")
    print("  builder: first loads", rel(t[0, 0, 5]), "chunk0 issued", rel(t[0, 0, 7]),
          "chunk1 issued", rel(t[0, 0, 8]), "prefetches issued", rel(t[0, 0, 6]),
          "loop top", rel(t[0, 0, 0]), "all stored", rel(t[0, 0, 1]))
    print("  set-up: barriers initialised", rel(t[6, 7, 0]), "TMEM allocated", rel(t[6, 7, 1]),
          "CTA barrier", rel(t[6, 7, 2]), "cluster barrier", rel(t[6, 7, 3]))
    print("  MMA: tile start", rel(t[2, 0, 0]), "G1 issued", rel(t[2, 0, 1]), "E1 seen", rel(t[2, 0, 3]))
    for c in range(6):
        print(f"  chunk {c}: slot free {rel(t[3, 0, c])}  stored {rel(t[4, 0, c])}  MMA saw {rel(t[5, 0, c])}")
    for k in range(8):
        print(f"  weight stage {k}: producer issued {rel(t[6, 0, k])}  MMA saw (next_b #{k}) {rel(t[7, 0, k])}")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "prologue":
    prologue(int(sys.argv[1]))
