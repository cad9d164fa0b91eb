# A/B of voxel edges/margins: args are "H MARGIN H2" triples.
mkdir -p gpurun_out
for v in "$@"; do
  set -- $v
  echo "variant h=$1 margin=$2 h2=$3" >> gpurun_out/ab_voxel.log
  GD_VOXEL_H=$1 GD_VOXEL_MARGIN=$2 GD_VOXEL_H2=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_voxel.log 2>&1
done
