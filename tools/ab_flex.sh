# A/B of flex-kernel build knobs on the GPU box (run from the repo root).
# Usage: bash tools/ab_flex.sh "RESIDENT_WARPS BATCH" ...   (BATCH 0 = chosen per launch)
mkdir -p gpurun_out
for v in "$@"; do
  set -- $v
  GD_NVCC_EXTRA="-DGD_FLEX_RESIDENT=$1 -DGD_FLEX_BATCH=${2:-0}" \
    python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
  echo "variant minb=$1 batch=${2:-0}" >> gpurun_out/ab_flex.log
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_flex.log 2>&1
done
python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
