"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the discriminator and the
synthetic image pool.

PARITY UNPINNED against the reference: the reference has no discriminator
network (SURVEY.md 8(c) row "Discriminator network (S9)"). This is
a restatement of THIS repo's PatchDisc definition (DESIGN.md
"Discriminator"): layer 1 as the exact integer GEMM the kernel runs (u8 pixels
x int8 weights, exact integer sums in fp64 here / s32 on the tensor cores --
identical values), then
fp32 numpy with the same bf16 rounding points as the GPU kernel (H1 and H2
are rounded to bf16 before the next GEMM), used to check
paper_2411_15381_b200/csrc/disc.cu within the north_star tolerance
(|dc| <= 1e-3 * max(|c|, 1e-2)). Accumulation order differs from the tensor
cores, so agreement is within tolerance, not bitwise.

synth_images() restates paper_2411_15381_b200/csrc/synth.cu byte for byte.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & M64
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return x ^ (x >> np.uint64(31))


def synth_images(seed: int, id0: int, n: int, h: int, w: int) -> np.ndarray:
    """Host restatement of ds_synth_images_device (synth.cu)."""
    with np.errstate(over="ignore"):
        smix = _splitmix64(np.array([seed], np.uint64))[0]
        nbytes = h * w * 3
        out = np.empty((n, nbytes), np.uint8)
        words = np.arange(nbytes // 8, dtype=np.uint64)
        for i in range(n):
            img_id = np.uint64(id0 + i)
            level = int(_splitmix64(np.array([smix ^ (~img_id & M64)], np.uint64))[0] >> np.uint64(56))
            r = _splitmix64(smix ^ ((img_id << np.uint64(24)) | words))
            b = r.view(np.uint8).astype(np.uint16)        # little-endian bytes of each word
            out[i] = ((b + level) >> 1).astype(np.uint8)
    return out.reshape(n, h, w, 3)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as f32."""
    u = x.astype(np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    return (0.5 * x * (1.0 + np.tanh(np.float32(0.7978845608028654) *
                                     (x + np.float32(0.044715) * x * x * x)))).astype(np.float32)


def patches(images: np.ndarray) -> np.ndarray:
    """(n,H,W,3) u8 -> (n, T, 768) f32; token t = py*(W/16)+px, k = dy*48+dx*3+c."""
    n, h, w, c = images.shape
    x = images.reshape(n, h // 16, 16, w // 16, 16, 3).transpose(0, 1, 3, 2, 4, 5)
    return x.reshape(n, (h // 16) * (w // 16), 768).astype(np.float32)


def disc_forward(images: np.ndarray, wts: dict, logits: bool = False) -> np.ndarray:
    q1 = wts["q1"].astype(np.float64)
    s1 = np.float32(wts["s1"])
    w2 = bf16_bits_to_f32(wts["w2"])
    w3 = bf16_bits_to_f32(wts["w3"])
    out = np.zeros(len(images), np.float32)
    for i in range(len(images)):
        x = patches(images[i:i + 1])[0].astype(np.float64)
        # the exact integer sums (|acc| <= 768*255*127 < 2^53: every fp64 partial
        # sum is an exact integer in any order, so BLAS dgemm is exact), then f32
        acc = (x @ q1).astype(np.float32)
        h1 = round_bf16(gelu_tanh(acc * s1 + wts["b1"]))
        h2 = round_bf16(np.maximum(h1 @ w2 + wts["b2"], 0.0))
        h3 = np.maximum(h2 @ w3 + wts["b3"], 0.0)
        s = h3 @ wts["head_w"]
        lg = np.float32(s.mean(dtype=np.float64)) + np.float32(wts["head_b"])
        out[i] = lg if logits else 1.0 / (1.0 + np.exp(-np.float64(lg)))
    return out


def disc_forward_fast(images: np.ndarray, wts: dict, threads: int = 0,
                      chunk: int = 1) -> np.ndarray:
    """disc_forward for TIMING (the bench's CPU baseline), as fast as numpy
    gets on the host: layer 1 in fp32 on CENTRED pixels (x - 128 in [-128,
    127], |q1| <= 127, so every partial sum is an integer below
    768*128*127 < 2^24 and exact in fp32 in any order: acc = (x-128) @ q1 +
    128 * colsum(q1), the same integers as the fp64 path), images in chunks
    of `chunk` per BLAS call, chunks spread over `threads` host threads with
    single-threaded BLAS in each (numpy's elementwise passes are single
    threaded; threads over chunks use every core for them too). Same values
    as disc_forward up to fp32 summation order in layers 2-3."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    q1 = wts["q1"].astype(np.float32)
    q1c = np.float32(128.0) * q1.astype(np.float64).sum(0).astype(np.float32)
    s1 = np.float32(wts["s1"])
    w2 = bf16_bits_to_f32(wts["w2"])
    w3 = bf16_bits_to_f32(wts["w3"])
    b1, b2, b3 = (np.asarray(wts[k], np.float32) for k in ("b1", "b2", "b3"))
    hw = np.asarray(wts["head_w"], np.float32)
    out = np.zeros(len(images), np.float32)
    t = len(images[0].reshape(-1)) // 768 if len(images) else 0

    def run(lo):
        hi = min(lo + chunk, len(images))
        x = patches(images[lo:hi]).reshape(-1, 768)
        x -= np.float32(128.0)
        acc = x @ q1
        acc += q1c
        h1 = round_bf16(gelu_tanh(acc * s1 + b1))
        h2 = round_bf16(np.maximum(h1 @ w2 + b2, 0.0))
        h3 = np.maximum(h2 @ w3 + b3, 0.0)
        sc = (h3 @ hw).reshape(hi - lo, t)
        for j in range(hi - lo):
            lg = np.float32(sc[j].mean(dtype=np.float64)) + np.float32(wts["head_b"])
            out[lo + j] = 1.0 / (1.0 + np.exp(-np.float64(lg)))

    threads = threads or (os.cpu_count() or 1)
    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(1, user_api="blas")
    except Exception:   # noqa: BLE001 -- without threadpoolctl BLAS oversubscribes
        limit = None
    try:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(0, len(images), chunk)))
    finally:
        if limit is not None:
            limit.restore_original_limits()
    return out


# ---- host restatement of the deterministic weights (disc.cu gen_weights_kernel,
# fold_bias_kernel and ds_disc_create's head) -------------------------------------

def _unif_pm1(stream: int, idx: np.ndarray) -> np.ndarray:
    """disc.cu unif_pm1: (splitmix64(stream ^ splitmix64(idx)) >> 11) * 2^-52 - 1, as f32."""
    with np.errstate(over="ignore"):
        r = _splitmix64(np.uint64(stream) ^ _splitmix64(idx.astype(np.uint64)))
    return ((r >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0).astype(np.float32)


def _to_bf16_bits(x: np.ndarray) -> np.ndarray:
    return (round_bf16(x).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def layer1_scale() -> np.float32:
    """disc.cu layer1_scale(): sqrt(3)/(64 sqrt(768)) / 127 in f32 arithmetic."""
    f32 = np.float32
    return (f32(1.7320508) / (f32(64.0) * f32(27.712812921102035))) / f32(127.0)


def gen_weights(seed: int, calibrate: bool = True) -> dict:
    """The PatchDisc weights ds_disc_create(seed) builds, restated on the host.
    Q1/s1, W2/W3 bits and b1 are bit-identical to the device; the head is
    calibrated here on the CPU forward pass (the device calibrates with its own
    logits, so head_w/head_b agree to ~1e-6 relative, see tests)."""
    f32 = np.float32
    s2 = f32(1.7320508) * np.sqrt(f32(2.0) / f32(256.0))
    s3 = f32(1.7320508) * np.sqrt(f32(2.0) / f32(1024.0))
    i1 = np.arange(768 * 256, dtype=np.uint64)
    # round-half-even of 127 u (f32 product), as __float2int_rn(__fmul_rn(127, u))
    q1 = np.rint(f32(127.0) * _unif_pm1(seed ^ 0x1111, i1)).astype(np.int8).reshape(768, 256)
    q1[:, 255] = 0
    s1 = layer1_scale()
    n2 = 256 * 1024
    e2 = np.arange(n2, dtype=np.uint64)
    w2f = s2 * _unif_pm1(seed ^ 0x2222, e2)
    w2f = w2f.reshape(256, 1024)
    w2f[255, :] = (f32(0.05) * _unif_pm1(seed ^ 0x5555, np.arange(1024, dtype=np.uint64))) / f32(16)
    w2f[:, 1023] = 0.0
    w2f[255, 1023] = 1.0
    w2 = _to_bf16_bits(w2f)
    e3 = np.arange(1024 * 256, dtype=np.uint64)
    w3f = (s3 * _unif_pm1(seed ^ 0x3333, e3)).reshape(1024, 256)
    w3f[1023, :] = (f32(0.05) * _unif_pm1(seed ^ 0x6666, np.arange(256, dtype=np.uint64))) / f32(16)
    w3 = _to_bf16_bits(w3f)
    # b1: exact integer column sums of Q1, then (-128 s1) * sum + 0.05 u with
    # separate f32 roundings
    col = q1.astype(np.int64).sum(axis=0).astype(np.float32)
    u4 = _unif_pm1(seed ^ 0x4444, np.arange(256, dtype=np.uint64))
    b1 = ((f32(-128.0) * s1) * col + f32(0.05) * u4).astype(np.float32)
    b1[255] = 16.0
    hw = (_unif_pm1(seed ^ 0x7777, np.arange(256, dtype=np.uint64)) / f32(16.0)).astype(np.float32)
    wts = dict(q1=q1, s1=float(s1), w2=w2, w3=w3, b1=b1, b2=np.zeros(1024, np.float32),
               b3=np.zeros(256, np.float32), head_w=hw, head_b=0.0)
    if calibrate:
        cal = synth_images(0xCA11B8A7E, 0, 64, 512, 512)
        lg = disc_forward(cal, wts, logits=True).astype(np.float64)
        mean = lg.mean()
        sd = np.sqrt(((lg - mean) ** 2).mean())
        scale = np.float32(2.0 / sd)
        wts["head_w"] = (hw * scale).astype(np.float32)
        wts["head_b"] = float(np.float32(-mean * scale))
    return wts
