"""TEST INFRASTRUCTURE ONLY -- a plain PyTorch fp32 reference of the
discriminator (PatchDisc, csrc/disc.cu header), written
independently of oracle/disc_oracle.py with torch ops: unfold into 16x16x3
patches, layer 1 as the exact integer GEMM of u8 pixels and int8 weights
(fp64 accumulate: every partial sum is an integer < 2^53), then fp32 with the
kernel's bf16 rounding of H1 and H2, ReLU, head mean and sigmoid."""
from __future__ import annotations

import numpy as np
import torch


def disc_forward_torch(images: np.ndarray, wts: dict) -> np.ndarray:
    x = torch.from_numpy(np.ascontiguousarray(images))                 # (n, H, W, 3) u8
    n, h, w, _ = x.shape
    # token t = py*(W/16)+px, feature k = dy*48 + dx*3 + c
    p = x.view(n, h // 16, 16, w // 16, 16, 3).permute(0, 1, 3, 2, 4, 5)
    p = p.reshape(n, (h // 16) * (w // 16), 768).to(torch.float64)
    q1 = torch.from_numpy(wts["q1"].astype(np.float64))
    acc = (p @ q1).to(torch.float32)                                    # exact s32 values
    s1 = torch.tensor(np.float32(wts["s1"]))
    b1 = torch.from_numpy(wts["b1"])
    h1 = torch.nn.functional.gelu(acc * s1 + b1, approximate="tanh")
    h1 = h1.to(torch.bfloat16).to(torch.float32)

    def bf16_weights(bits):
        return torch.from_numpy((bits.astype(np.uint32) << 16).view(np.float32).copy())
    w2, w3 = bf16_weights(wts["w2"]), bf16_weights(wts["w3"])
    h2 = torch.relu(h1 @ w2 + torch.from_numpy(wts["b2"])).to(torch.bfloat16).to(torch.float32)
    h3 = torch.relu(h2 @ w3 + torch.from_numpy(wts["b3"]))
    s = h3 @ torch.from_numpy(wts["head_w"])                            # (n, T)
    logit = s.to(torch.float64).mean(dim=1) + float(wts["head_b"])
    return torch.sigmoid(logit).numpy()
