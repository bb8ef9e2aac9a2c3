#!/bin/bash
# K3 on the GPU box: curve parity tests, then replay timings at the bench sizes
# (5K: the image step; 32K: the smallest segmented replay; 1M: the latent leg),
# with the single-CTA replay beside them (DS_CURVE_SPEC=0).
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_score_route.py -x -q -k curve 2>&1 | tail -5
for n in 5000 32768 1000000; do
    timeout 120 python tools/curve_speed.py $n
    DS_CURVE_SPEC=0 timeout 120 python tools/curve_speed.py $n
done
