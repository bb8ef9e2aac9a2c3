#!/bin/bash
# A/B kernel variants on the GPU box: for each argument (a set of -D flags, or
# "default"), rebuild libds_b200.so with DS_EXTRA_NVCC and time the kernel.
#   tools/ab.sh default "-DFOO=1" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
    if [ "$v" = default ]; then unset DS_EXTRA_NVCC; else export DS_EXTRA_NVCC="$v"; fi
    python -c "from paper_2411_15381_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
    for r in 1 2; do timeout 120 python tools/${AB_TOOL:-disc_speed.py}; done
done
unset DS_EXTRA_NVCC
python -c "from paper_2411_15381_b200 import build; build.build(force=True)" > /dev/null 2>&1
