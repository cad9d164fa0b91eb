for v in "GD_VOXEL_H2=0.75" "GD_VOXEL_H2=1.0" "GD_VOXEL_H2=1.25" "GD_VOXEL_H2=1.0 GD_VOXEL_MARGIN2=16" "GD_VOXEL_H2=1.5 GD_VOXEL_MARGIN2=24"; do
  echo "== $v"; env $v python tools/quick_bench.py --configs 1 2 --reps 3
done
