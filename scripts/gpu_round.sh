#!/usr/bin/env bash
# One GPU call: parity tests, the default bench line (both arms), the launch
# list of the production step at 16.4M and a full ncu capture of the fused
# step kernel (each ncu pass only after its command exited 0 without ncu).
# TAG=r02a bash scripts/gpu_round.sh [skip-tests]
set -u
TAG=${TAG:-r02a}
mkdir -p gpurun_out
if [ "${1:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench_ref.json
if timeout 600 python scripts/prof_step.py 160 30 > gpurun_out/${TAG}_prof_step.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_160.csv python scripts/prof_step.py 160 30 \
      > gpurun_out/${TAG}_ncu_launches.log 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forces_l1 -s 12 -c 1 \
      -o gpurun_out/${TAG}_step_kernel python scripts/prof_step.py 160 30 > gpurun_out/${TAG}_ncu_step.log 2>&1
  echo "ncu full rc=$?"
else
  echo "prof_step failed"; tail -20 gpurun_out/${TAG}_prof_step.log
fi
echo done
