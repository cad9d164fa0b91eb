# Full ncu capture of the flex and rigid kernels of one bench step (run from
# the repo root on the GPU box, after the same bench command exited 0).
# Usage: [KERNELS="flex_chain"] bash tools/prof.sh TAG
mkdir -p gpurun_out
python paper_1901_06363_b200/build.py > /dev/null
for k in ${KERNELS:-flex_chain rigid_top}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-1} -c 1 \
    -o gpurun_out/prof_${1}_${k} -f \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_${1}_${k}.log 2>&1
done
