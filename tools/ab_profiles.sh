# A/B of -D build variants on the analysis workload (bench.py --workload profiles).
mkdir -p gpurun_out
for v in "$@"; do
  GD_DEFS="$v" python paper_1901_06363_b200/build.py --force > /dev/null 2>&1 || { echo "variant $v BUILD FAILED"; continue; }
  echo "variant $v"
  python bench.py --workload profiles --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['kernel_ms'])"
done
python paper_1901_06363_b200/build.py --force > /dev/null 2>&1
