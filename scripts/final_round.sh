#!/usr/bin/env bash
# End-of-round evidence on the final build, one GPU call: the GPU suite, the
# driver's bench command (both arms), the other configs, and the launch list
# of the bench command itself (eager: TMD_GRAPHS=0, ncu cannot profile the
# kernel nodes of graphs with conditional nodes) after it ran clean without ncu.
set -u
TAG=${TAG:-r02y}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
run() { local name=$1; shift; timeout 1200 "$@" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err || echo "$name failed"; tail -c 300 gpurun_out/${TAG}_${name}.json; echo; }
run bench python bench.py --steps 20 --warmup 5
run bench_ref python bench.py --impl reference --steps 20 --warmup 5
run bench_steady python bench.py --steps 500 --warmup 10 --no-cpu-baseline
run bench_cells64 python bench.py --cells 64 --steps 1000 --no-cpu-baseline
run bench_cells20 python bench.py --cells 20 --steps 2000 --no-cpu-baseline
run bench_kg python bench.py --config kg --cells 64 --steps 1000 --no-cpu-baseline
run bench_slab python bench.py --config slab --cells 64 --steps 1000 --no-cpu-baseline
if TMD_GRAPHS=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_eager.json 2> gpurun_out/${TAG}_bench_eager.err; then
  TMD_GRAPHS=0 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/${TAG}_bench_launches.csv \
      python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
fi
echo done
