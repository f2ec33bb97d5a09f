#!/bin/bash
# Profile evidence for profiles/ (run under gpurun on one B200).  Every ncu command is
# preceded by the same command without ncu, which must exit 0 first.
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
$BENCH > "$OUT/bench_plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_bench.csv" \
    $BENCH > "$OUT/ncu_launches.log" 2>&1
PROF="python tools/prof_run.py --n 30 --p 4"
$PROF > "$OUT/prof_plain.log" 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tma_ -s 1 -c 3 \
    -o "$OUT/tma_pass_full" $PROF > "$OUT/ncu_full.log" 2>&1
echo done
