# Round measurement batch (one gpurun call): small-problem probe, per-config probe, cfg3 sweep,
# bench (both arms).  Outputs under gpurun_out/ with the tag given as $1.
T=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
python tools/small_probe.py 1 abc 2 abc 0 abc 1 ab 2 ab > gpurun_out/${T}_small.txt 2>&1
python tools/kernel_timeline.py cfg1 1 abc 2>/dev/null | tail -6 >> gpurun_out/${T}_small.txt
python tools/perf_probe.py cfg1 cfg2 cfg4 bar cfg5s8 cfg5 > gpurun_out/${T}_perf_probe.txt 2>&1
python tools/cfg3_sweep.py > gpurun_out/${T}_cfg3_sweep.txt 2>&1
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
tail -3 gpurun_out/${T}_*.txt; cat gpurun_out/${T}_bench.json
