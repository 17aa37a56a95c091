#!/usr/bin/env bash
# Quick GPU status check: full GPU suite + bench lines at the default, 1M and 32K.
set -u
TAG=${TAG:-r02n}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest_gpu.log
run() { local name=$1; shift; timeout 900 "$@" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err || echo "$name failed"; tail -c 600 gpurun_out/${TAG}_${name}.json; echo; }
run bench python bench.py --steps 20 --warmup 5
run bench_cells64 python bench.py --cells 64 --steps 1000 --no-cpu-baseline
run bench_cells20 python bench.py --cells 20 --steps 2000 --no-cpu-baseline
TMD_SPEC=0 timeout 600 python bench.py --cells 20 --steps 2000 --no-cpu-baseline > gpurun_out/${TAG}_bench_cells20_nospec.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_cells20_nospec.json
TMD_SPEC=0 timeout 600 python bench.py --cells 64 --steps 1000 --no-cpu-baseline > gpurun_out/${TAG}_bench_cells64_nospec.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_cells64_nospec.json
timeout 300 python scripts/exp/speclog.py > gpurun_out/${TAG}_speclog.log 2>&1; tail -20 gpurun_out/${TAG}_speclog.log
echo done
