# A/B of runtime environment variants (e.g. GD_VOXEL_H=0.2) on the GPU box.
# Usage: bash tools/ab_env.sh "VAR=val VAR2=val" ...   ("" = defaults)
mkdir -p gpurun_out
python paper_1901_06363_b200/build.py > /dev/null 2>&1
for v in "$@"; do
  echo "variant env $v" >> gpurun_out/ab_defs.log
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_defs.log 2>&1
done
