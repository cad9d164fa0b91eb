# A/B of the flex kernel's shared-memory carveout (percent of 228 KB).
mkdir -p gpurun_out
for c in "$@"; do
  echo "variant carveout=$c" >> gpurun_out/ab_carveout.log
  GD_FLEX_CARVEOUT=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_carveout.log 2>&1
done
