#!/bin/bash
# Round-end measurement package (run under gpurun): bench record, ncu launch list of the same command,
# ncu --set full capture of the matvec kernels.  Each ncu pass only after the same command exited 0 without ncu.
set -e
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-bie --no-cfg4 --no-deterministic"
$B > gpurun_out/final_bench_short.json 2> /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launch_list.csv $B > gpurun_out/final_ncu_launch.log 2>&1
python scripts/profile_matvec.py cfg2 1048576 1 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:"translate64|p2p_kernel|p2m_fast|l2p_fast" -o gpurun_out/final_cfg2_full python scripts/profile_matvec.py cfg2 1048576 1 > gpurun_out/final_ncu_full.log 2>&1
tail -c 400 gpurun_out/final_bench.json
