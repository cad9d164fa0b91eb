# ncu captures of the flex and rigid kernels with the fp64 and the coded
# voxel-record formats (run on the GPU box from the repo root).
# Usage: bash tools/prof_fmt.sh TAG
mkdir -p gpurun_out
for f in 0 1; do
  GD_INDEX_COMPACT=$f timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_${1}_fmt${f}_bench.json 2>&1 || exit 1
  for k in flex_chain rigid_top; do
    GD_INDEX_COMPACT=$f timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_${1}_fmt${f}_${k} -f \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_${1}_fmt${f}_${k}.log 2>&1
  done
done
