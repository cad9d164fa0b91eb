#!/bin/bash
# A/B of source variants of one CUDA file on the GPU box (repo root).
# Usage: bash tools/ab_src.sh csrc/flex.cu ab_variants/flex_A.cu ab_variants/flex_B.cu ...
# Runs the variants interleaved twice (A B .. A B ..), 5 timed steps each,
# and restores the original file afterwards.
mkdir -p gpurun_out
target=paper_1901_06363_b200/$1; shift
cp "$target" /tmp/ab_src_orig
for round in 1 2; do
  for v in "$@"; do
    cp "$v" "$target"
    if ! python paper_1901_06363_b200/build.py > /dev/null 2>&1; then
      echo "variant $v BUILD FAILED" >> gpurun_out/ab_src.log; continue
    fi
    echo "variant $v round $round" >> gpurun_out/ab_src.log
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_src.log 2>&1
  done
done
cp /tmp/ab_src_orig "$target"
python paper_1901_06363_b200/build.py > /dev/null 2>&1
