#!/bin/bash
# r02 A/B sweep: fused GAT (U, CTAs/SM) x score block; weighted-reverse alpha L2 policy; edge scales
mkdir -p gpurun_out
out=gpurun_out/sweep.txt
: > $out
for t in 0 1 2 3; do
  for kb in 3 4 5 7; do
    echo "GAT tune=$t smem_kb=$kb $(GSP_TUNE_GAT=$t GSP_GAT_SMEM_KB=$kb timeout 120 python tools/opbench.py --ops gat_fused --reps 7 2>&1 | tail -1)" >> $out
  done
done
for p in 0 1 2; do
  for w in 1024 2048 4096; do
    echo "WREV pol=$p win=$w $(GSP_WREV_POL=$p GSP_EID_WIN=$w timeout 120 python tools/opbench.py --ops wrev --reps 7 2>&1 | tail -1)" >> $out
  done
done
timeout 600 python tools/ab_edge_scales.py --out gpurun_out/ab_edge_scales.json > gpurun_out/ab_edge_scales.log 2>&1
cat $out
