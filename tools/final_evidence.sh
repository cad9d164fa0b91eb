# End-of-round evidence on the GPU box (repo root): bench lines, reference arm,
# analysis bench, launch list, full ncu captures, config-4 sweep, configs 2 and 3.
# Edit the tag (r2j) per round.
python paper_1901_06363_b200/build.py --force > /dev/null
python bench.py > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2j_ref.json 2> gpurun_out/bench_r2j_ref.err
python bench.py --workload profiles > gpurun_out/bench_r2j_prof.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2j.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
bash tools/prof.sh r2j
timeout 2400 python tools/knob_sweep.py --ligands 20000 --pockets 4 --full > gpurun_out/knob_sweep_full_r2j.json 2> gpurun_out/knob_sweep_full_r2j.err
python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_r2j_c2.json 2>&1
timeout 900 python tools/screen_c3.py > gpurun_out/c3_r2j.json 2> gpurun_out/c3_r2j.err
