# A/B of rigid-kernel build knobs on the GPU box (run from the repo root).
# Usage: bash tools/ab_rigid.sh "MINB MLP" ...
mkdir -p gpurun_out
for v in "$@"; do
  set -- $v
  GD_NVCC_EXTRA="-DGD_RIGID_MINB=$1 -DGD_RIGID_MLP=$2" \
    python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
  echo "variant rigid minb=$1 mlp=$2" >> gpurun_out/ab_rigid.log
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_rigid.log 2>&1
done
python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
