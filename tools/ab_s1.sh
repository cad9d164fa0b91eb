# Same-box A/B of the voxel-record formats (fp64 vs coded) on configs 1 and 2,
# after the index-format and parity tests.  Usage: bash tools/ab_s1.sh
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_index_formats.py tests/test_gpu_parity.py -x -q > gpurun_out/s1_tests.log 2>&1
for r in 1 2; do
for v in GD_INDEX_COMPACT=0 GD_INDEX_COMPACT=1; do
  echo "variant $v" >> gpurun_out/s1_ab.log
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/s1_ab.log 2>&1
  env $v timeout 300 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/s1_ab.log 2>&1
done
done
