#!/usr/bin/env bash
# Full ncu captures of the brick kernels: the first (setup) list build, and two
# steady-state force launches. Plain run first (must exit 0).
set -u
CMD=${CMD:-"python bench.py --steps 30 --warmup 3 --no-cpu-baseline"}
TAG=${TAG:-r01b}
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-700} --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"${BUILDK:-k_build_brick}" -s 0 -c 1 \
    -o gpurun_out/prof_build_${TAG} $CMD > gpurun_out/ncu_build.log 2>&1
echo "build capture rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"${FORCEK:-k_forces_brick}" -s 10 -c 1 \
    -o gpurun_out/prof_force_${TAG} $CMD > gpurun_out/ncu_force.log 2>&1
echo "force capture rc=$?"
