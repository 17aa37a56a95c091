#!/usr/bin/env bash
# Profiling recipe (run under gpurun, one GPU). Plain run first; ncu only if it
# exited 0 (B200_PROFILING.md). Outputs land in gpurun_out/.
set -u
CMD=${CMD:-"python bench.py --steps 30 --warmup 3 --no-cpu-baseline"}
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
if [ "${LAUNCHES:-1}" = 1 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-600} --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
  echo "launch list rc=$?"
fi
if [ -n "${FULL:-}" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"${FULL}" -s ${SKIP:-5} -c ${COUNT:-2} \
      -o gpurun_out/prof_${TAG:-r01} $CMD > gpurun_out/ncu_full.log 2>&1
  echo "full capture rc=$?"
fi
