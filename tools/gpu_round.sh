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
if [ -n "$L2BENCH" ] && [ -x tools/l2bench ]; then
  (tools/l2bench 232965; tools/l2bench 116483) > gpurun_out/l2bench.txt 2>&1
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --profile --steps 2 --warmup 1 > gpurun_out/launches_bench.log 2>&1
  # the timed step of the default (fused GAT chain) bench: 4 kernels after the warm-up step's 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm|softmax|gat_fused" -s 4 -c 4 \
      -o gpurun_out/prof_step python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
  # the separate chain (gSDDMM, softmax, weighted fwd as their own kernels): 6 after 6
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm|softmax" -s 6 -c 6 \
      -o gpurun_out/prof_step_sep python bench.py --profile --chain separate --steps 1 --warmup 1 > gpurun_out/ncu_full_sep.log 2>&1
  # ogbn-products-shaped gSpMM (DRAM-resident 980 MB table): the timed step's fwd + rev launches
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm" -s 2 -c 2 \
      -o gpurun_out/prof_products python bench.py --config products --profile --steps 1 --warmup 1 > gpurun_out/ncu_products.log 2>&1
  [ -f gpurun_out/prof_products.ncu-rep ] && ncu -i gpurun_out/prof_products.ncu-rep --page raw --csv > gpurun_out/prof_products.raw.csv 2>/dev/null
  rm -f gpurun_out/prof_products.ncu-rep
  # Reddit F = 602 (561 MB table, ld 604) and ogbn-arxiv F = 128: one gSpMM fwd launch each, after opbench's 3 warm-ups
  timeout 600 ncu --set full --clock-control none -k regex:"spmm" -s 3 -c 1 -o gpurun_out/prof_f602 \
      python tools/opbench.py --F 602 --ld 604 --ops gspmm_fwd --reps 1 > gpurun_out/ncu_f602.log 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:"spmm" -s 3 -c 1 -o gpurun_out/prof_arxiv \
      python tools/opbench.py --config arxiv --ops gspmm_fwd --reps 1 > gpurun_out/ncu_arxiv.log 2>&1
  for r in prof_f602 prof_arxiv; do
    [ -f gpurun_out/$r.ncu-rep ] && ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
    rm -f gpurun_out/$r.ncu-rep
  done
  # gpurun copies back <= 64 MiB: raw csv of both captures, drop the separate-chain report
  for r in prof_step prof_step_sep; do
    [ -f gpurun_out/$r.ncu-rep ] && ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
  done
  rm -f gpurun_out/prof_step_sep.ncu-rep
fi
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.json
