# Same-box A/B of whole source trees (git worktrees under ab_variants/),
# interleaved repeats.  Usage: bash tools/ab_trees.sh REPS tree1 tree2 ...
# ("." = the repo itself).  Appends to gpurun_out/ab_trees.log.
mkdir -p gpurun_out
reps=$1; shift
for r in $(seq 1 $reps); do
  for t in "$@"; do
    echo "tree $t rep $r" >> gpurun_out/ab_trees.log
    (cd $t && timeout 300 python tools/quick_bench.py --configs ${AB_CONFIGS:-1 2} --reps 3) >> gpurun_out/ab_trees.log 2>&1
  done
done
