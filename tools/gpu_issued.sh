#!/bin/bash
# Issued fp64 / fp32 FMA and DMMA work of the evaluator kernels (SURVEY 8(d) "issued FMA fraction"), cfg3 and
# cfg5-fp32: explicit counters, one ncu pass each (after the same command ran without ncu).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M="gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__ops_path_tensor_src_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"
for spec in "3:" "5:--fp32"; do
  cfg=${spec%%:*}; extra=${spec#*:}; tag=cfg${cfg}${extra:+_fp32}
  C="python tools/run_cfg.py --config $cfg $extra --steps 2"
  $C > /dev/null 2>&1 && timeout 900 ncu --metrics $M --clock-control none -k regex:"k_eval" --csv --log-file gpurun_out/issued_$tag.csv $C > /dev/null 2>&1
done
