# e2e chunk-plan A/B (repo root, GPU box): bash tools/e2e_ab.sh "GD_E2E_HEAD=256 GD_E2E_CHUNKS=15" ...
mkdir -p gpurun_out
python paper_1901_06363_b200/build.py > /dev/null 2>&1
for v in "$@"; do
  echo "variant $v" >> gpurun_out/e2e_ab.log
  env $v timeout 300 python tools/e2e_probe.py 2>&1 | tail -3 >> gpurun_out/e2e_ab.log
done
