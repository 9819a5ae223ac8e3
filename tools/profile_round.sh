#!/usr/bin/env bash
# Evidence pass for a round (run under gpurun on ONE GPU):
#   tools/profile_round.sh <tag>
# writes gpurun_out/<tag>/: bench.json (the driver's command), launches.csv
# (every launch of a short bench run with its device time), metrics.csv
# (DRAM bytes / L2 atomics of the step kernels), full.ncu-rep (ncu --set full
# of the dominant bench kernel), probe.txt (all configs, per-task device time
# and top kernels).  Never a bench number from an ncu run.
# The bench's first warm-up step runs over the whole DAG and builds the
# single-parent contraction (contract.cu); the metric and --set full passes
# skip it (-s) and stop before the e2e repetitions, which open fresh DAGs.
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
cp paper_2106_06889_b200/_build/stamp "$OUT/stamp.txt" 2>/dev/null
timeout 400 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"k_segred|k_seed|k_root_words|k_expand_rows|k_popc_rows|k_records|k_ii_groups" -s 1 -c 4 --csv \
  --log-file "$OUT/metrics.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_segred1?_levels" -s 2 -c 1 \
  -o "$OUT/full" python bench.py --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/full.log" 2>&1
timeout 900 python tools/gpu_probe.py c2 c3 c4 c5 --pinned --reps 4 > "$OUT/probe.txt" 2>&1
GT_TRACE=2 timeout 300 python tools/step_probe.py c2 --reps 4 > "$OUT/step_phases.txt" 2>&1
GT_TRACE=2 timeout 300 python tools/gpu_probe.py c2 c5 --pinned --tasks wordcount --reps 1 > "$OUT/open_trace.txt" 2>&1
echo done
