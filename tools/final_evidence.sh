# End-of-round evidence on the GPU box (repo root): bench lines, reference arm,
# analysis bench, launch list, full ncu captures, config-4 sweep.
python paper_1901_06363_b200/build.py --force > /dev/null
python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2e_ref.json 2> gpurun_out/bench_r2e_ref.err
python bench.py --workload profiles > gpurun_out/bench_r2e_prof.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2e.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
bash tools/prof.sh r2e
timeout 2400 python tools/knob_sweep.py --ligands 20000 --pockets 4 --full > gpurun_out/knob_sweep_full_r2.json 2> gpurun_out/knob_sweep_full_r2.err
