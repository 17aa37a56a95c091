#!/usr/bin/env bash
# Round-2 evidence in one GPU call: bench lines of every BASELINE config (our
# arm; the reference arm for the default), eager launch lists with DRAM bytes
# at 16.4M and 32K, and full ncu captures of the fused step kernel and the
# list build at 16.4M (each ncu pass after its command ran clean without ncu).
set -u
TAG=${TAG:-r02t}
mkdir -p gpurun_out
run() { local name=$1; shift; timeout 1200 "$@" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err || echo "$name failed"; tail -c 400 gpurun_out/${TAG}_${name}.json; echo; }
run bench python bench.py --steps 20 --warmup 5
run bench_ref python bench.py --impl reference --steps 20 --warmup 5
run bench_steady python bench.py --steps 500 --warmup 10 --no-cpu-baseline
run bench_cells64 python bench.py --cells 64 --steps 1000 --no-cpu-baseline
run bench_cells20 python bench.py --cells 20 --steps 2000 --no-cpu-baseline
run bench_kg python bench.py --config kg --cells 64 --steps 1000 --no-cpu-baseline
run bench_slab python bench.py --config slab --cells 64 --steps 1000 --no-cpu-baseline
if timeout 600 python scripts/prof_step.py 160 30 > gpurun_out/${TAG}_prof_step160.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_160.csv python scripts/prof_step.py 160 30 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forces_l1 -s 12 -c 1 \
      -o gpurun_out/${TAG}_step_kernel python scripts/prof_step.py 160 30 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_cull -s 31 -c 1 \
      -o gpurun_out/${TAG}_build python scripts/prof_step.py 160 30 > /dev/null 2>&1
fi
if timeout 600 python scripts/prof_step.py 20 300 > gpurun_out/${TAG}_prof_step20.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_20.csv python scripts/prof_step.py 20 300 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forces_lanes -s 100 -c 1 \
      -o gpurun_out/${TAG}_step_kernel20 python scripts/prof_step.py 20 300 > /dev/null 2>&1
fi
timeout 300 python scripts/small_probe.py 20 > gpurun_out/${TAG}_small_probe.log 2>&1
timeout 300 python scripts/build_probe.py 20 64 160 > gpurun_out/${TAG}_build_probe.log 2>&1
timeout 300 python scripts/slab_overhead_probe.py 64 > gpurun_out/${TAG}_slab_overhead64.log 2>&1
timeout 300 python scripts/slab_overhead_probe.py 20 > gpurun_out/${TAG}_slab_overhead20.log 2>&1
timeout 300 python scripts/small_probe2.py 20 > gpurun_out/${TAG}_small_probe2.log 2>&1
timeout 300 python scripts/force_variants.py --cells 64 --steps 50 --variants 2,3:4 > gpurun_out/${TAG}_force_variants64.log 2>&1
echo done
