# A/B of -D build variants on a given bench config (repo root, GPU box).
# Usage: bash tools/ab_defs_cfg.sh CONFIG "-DA=1" "-DB=2" ...
mkdir -p gpurun_out
cfg=$1; shift
for v in "$@"; do
  if ! GD_DEFS="$v" python paper_1901_06363_b200/build.py --force > /dev/null 2>&1; then
    echo "variant $v BUILD FAILED" >> gpurun_out/ab_defs.log; continue
  fi
  echo "variant c$cfg $v" >> gpurun_out/ab_defs.log
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e >> gpurun_out/ab_defs.log 2>&1
done
python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
