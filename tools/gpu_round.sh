#!/bin/bash
# one GPU session: tests, bench, launch list and a full ncu capture of one step's kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m "${MARK:-gpu}" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --profile --steps 2 --warmup 1 > gpurun_out/launches_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm|softmax" -s 2 -c 6 \
      -o gpurun_out/prof_step python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.json
