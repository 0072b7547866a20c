#!/bin/bash
# Round-end evidence in one gpurun call: smoke, GPU tests, both bench arms, per-config probe,
# then (after the plain runs exited 0) the ncu launch list of the bench command and one
# --set full capture of the headline kernels.  Outputs under gpurun_out/ with tag $1.
T=${1:-final}
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py smoke
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
} > gpurun_out/${T}_validate.txt 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err || exit 1
python tools/perf_probe.py cfg1 cfg2 cfg4 bar cfg5s8 > gpurun_out/${T}_perf_probe.txt 2>&1
python tools/small_probe.py 1 abc 2 abc > gpurun_out/${T}_small.txt 2>&1
python bench.py --steps 2 --warmup 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/${T}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_strassen_fused|k_presum" -c 2 -o gpurun_out/prof_${T}_cfg5_L2_abc -f \
  python tools/one_call.py cfg5 2 abc 1 > gpurun_out/${T}_ncu_full.log 2>&1
tail -4 gpurun_out/${T}_validate.txt; tail -c 400 gpurun_out/${T}_bench.json
