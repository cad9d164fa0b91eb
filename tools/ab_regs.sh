mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "8 4" "6 4" "6 3" "5 3"; do
  set -- $v
  GD_NVCC_EXTRA="-DGD_FLEX_RESIDENT=$1 -DGD_RIGID_MINB=$2" python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
  echo "variant flex=$1 rigid=$2" >> gpurun_out/ab.log
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab.log 2>&1
done
