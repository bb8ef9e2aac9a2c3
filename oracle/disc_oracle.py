"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the discriminator and the
synthetic image pool.

PARITY UNPINNED against the reference: the reference has no discriminator
network (SURVEY.md 8(c) row "Discriminator network (S9)"). This is
a restatement of THIS repo's PatchDisc definition (DESIGN.md
"Discriminator"), in fp32 numpy with the same bf16 rounding points as the GPU
kernel (H1 and H2 are rounded to bf16 before the next GEMM), used to check
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
    w1 = bf16_bits_to_f32(wts["w1"])
    w2 = bf16_bits_to_f32(wts["w2"])
    w3 = bf16_bits_to_f32(wts["w3"])
    out = np.zeros(len(images), np.float32)
    for i in range(len(images)):
        x = patches(images[i:i + 1])[0]
        h1 = round_bf16(gelu_tanh(x @ w1 + wts["b1"]))
        h2 = round_bf16(np.maximum(h1 @ w2 + wts["b2"], 0.0))
        h3 = np.maximum(h2 @ w3 + wts["b3"], 0.0)
        s = h3 @ wts["head_w"]
        lg = np.float32(s.mean(dtype=np.float64)) + np.float32(wts["head_b"])
        out[i] = lg if logits else 1.0 / (1.0 + np.exp(-np.float64(lg)))
    return out
