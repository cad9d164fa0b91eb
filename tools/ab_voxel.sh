# A/B of the fine voxel edge (GD_VOXEL_H) on the GPU box.
mkdir -p gpurun_out
for h in "$@"; do
  echo "variant h=$h" >> gpurun_out/ab_voxel.log
  GD_VOXEL_H=$h timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_voxel.log 2>&1
done
