#!/usr/bin/env bash
# One GPU call that refreshes the round's evidence (run under gpurun):
# bench lines of every BASELINE config, the eager launch list with DRAM bytes,
# and full ncu captures of the list build and the fused force kernel (each ncu
# pass only after the same command exited 0 without ncu).
set -u
TAG=${TAG:-r01g}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || echo "bench failed"
for c in kg slab; do
  python bench.py --config $c > gpurun_out/${TAG}_bench_config$c.json 2> gpurun_out/${TAG}_bench_config$c.err || echo "bench $c failed"
done
python bench.py --cells 20 > gpurun_out/${TAG}_bench_cells20.json 2> gpurun_out/${TAG}_bench_cells20.err || echo "bench cells20 failed"
python bench.py --cells 160 --steps 500 > gpurun_out/${TAG}_bench_cells160.json 2> gpurun_out/${TAG}_bench_cells160.err || echo "bench cells160 failed"
if python scripts/prof_force.py 64 > gpurun_out/${TAG}_prof_plain.log 2>&1; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_eager.csv python scripts/prof_force.py 64 \
      > gpurun_out/${TAG}_ncu_launches.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_build_cull -s 51 -c 1 \
      -o gpurun_out/${TAG}_build python scripts/prof_force.py 64 > gpurun_out/${TAG}_ncu_build.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_forces_l1 -s 30 -c 1 \
      -o gpurun_out/${TAG}_force python scripts/prof_force.py 64 > gpurun_out/${TAG}_ncu_force.log 2>&1
fi
# the small-system force kernel (k_forces_lanes, configs[0])
if python scripts/prof_force.py 20 > gpurun_out/${TAG}_prof_plain20.log 2>&1; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_eager_32k.csv python scripts/prof_force.py 20 \
      > gpurun_out/${TAG}_ncu_launches32k.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_forces_lanes -s 30 -c 1 \
      -o gpurun_out/${TAG}_force_lanes python scripts/prof_force.py 20 > gpurun_out/${TAG}_ncu_force_lanes.log 2>&1
fi
echo done
