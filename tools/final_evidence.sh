# End-of-round evidence on the GPU box (repo root): bench lines, reference arm,
# analysis bench, launch list, full ncu captures, config-4 sweep, configs 2 and 3.
# Usage: bash tools/final_evidence.sh TAG   (e.g. r3a)
T=${1:?tag}
python paper_1901_06363_b200/build.py --force > /dev/null
python bench.py > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err
GD_HOST_THREADS=2 python bench.py --no-cpu-baseline > gpurun_out/bench_${T}_2threads.json 2> gpurun_out/bench_${T}_2threads.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
python bench.py --workload profiles > gpurun_out/bench_${T}_prof.json 2>&1
python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_${T}_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${T}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
bash tools/prof.sh ${T}
SKIP=0 KERNELS="prep_kernel" bash tools/prof.sh ${T}
timeout 900 python tools/screen_c3.py > gpurun_out/c3_${T}_multi.json 2> gpurun_out/c3_${T}_multi.err
timeout 900 python tools/screen_c3.py --ranks > gpurun_out/c3_${T}_ranks.json 2> gpurun_out/c3_${T}_ranks.err
timeout 2400 python tools/knob_sweep.py --ligands 20000 --pockets 4 --full > gpurun_out/knob_sweep_full_${T}.json 2> gpurun_out/knob_sweep_full_${T}.err
python tools/index_build_c3.py > gpurun_out/index_c3_${T}.txt 2>&1
