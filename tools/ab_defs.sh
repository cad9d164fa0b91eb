# A/B of -D build variants (applied to device and host objects) on the GPU
# box, from the repo root.  Usage: bash tools/ab_defs.sh "-DA=1 -DB=2" ...
mkdir -p gpurun_out
for v in "$@"; do
  if ! GD_DEFS="$v" python paper_1901_06363_b200/build.py --force > /dev/null 2>&1; then
    echo "variant $v BUILD FAILED" >> gpurun_out/ab_defs.log; continue
  fi
  echo "variant $v" >> gpurun_out/ab_defs.log
  timeout 300 python tools/quick_bench.py --configs ${AB_CONFIGS:-1 2} >> gpurun_out/ab_defs.log 2>&1
done
python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
