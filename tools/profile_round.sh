#!/bin/bash
# Round measurement pass (run under gpurun from the repo root): the bench line, the reference
# (oracle) arm, the ncu launch list of the same bench command, and one ncu --set full capture of
# every kernel of one view. Outputs land in gpurun_out/ ; tools/ncu_summary.py turns them into
# the committed profiles/ summaries.
set -u
R=${1:-r02}
mkdir -p gpurun_out
python -c "from paper_2504_12811_b200 import _build; _build.build()"
timeout 900 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
tail -3 gpurun_out/bench_${R}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${R}.json 2> gpurun_out/bench_ref_${R}.err
tail -3 gpurun_out/bench_ref_${R}.err
# launch list: per-launch durations of a short run of the same bench command (cold cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv \
    python bench.py --steps 2 --warmup 3 --scaling weak --views-per-rank 4 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_launch_${R}.err
tail -3 gpurun_out/ncu_launch_${R}.err
# full capture of one whole view (the 2nd rendered view: skip the load kernel + the first view)
timeout 1200 ncu --set full --metrics sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_lsu.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum --clock-control none --import-source on -k regex:^k_ -s 15 -c 15 \
    -o gpurun_out/full_${R} -f \
    python bench.py --steps 1 --warmup 3 --scaling weak --views-per-rank 1 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_full_${R}.err
tail -3 gpurun_out/ncu_full_${R}.err
ncu -i gpurun_out/full_${R}.ncu-rep --page raw --csv > gpurun_out/full_${R}_raw.csv 2>/dev/null
ls -la gpurun_out/
