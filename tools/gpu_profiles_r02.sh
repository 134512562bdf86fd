#!/bin/bash
# Round-2 evidence for profiles/: the bench line, the launch list of the bench command (cold-cache,
# serialised per-launch times), ncu --set full of every cfg3 kernel, the fp32 / real / sparse evaluators
# and the full-Horner context kernel.  Each ncu pass runs after the same command exited 0 without ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_cfg3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
C3="python tools/run_cfg.py --config 3 --steps 2"
$C3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 8 -c 8 -o /tmp/prof_cfg3_all $C3 > gpurun_out/ncu_cfg3_all.log 2>&1
python tools/summarize_ncu.py /tmp/prof_cfg3_all.ncu-rep > gpurun_out/r02_ncu_cfg3_all_kernels.json
for k in k_eval_tiled k_eval_mma k_classify_bucket k_bucket_scatter k_unsort; do python tools/ncu_hotlines.py /tmp/prof_cfg3_all.ncu-rep $k 25 >> gpurun_out/r02_ncu_cfg3_hotlines.txt; done
for spec in "5:--fp32" "2:" "4:"; do
  cfg=${spec%%:*}; extra=${spec#*:}; tag=cfg${cfg}${extra:+_fp32}
  C="python tools/run_cfg.py --config $cfg $extra --steps 2"
  $C > gpurun_out/plain_$tag.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_classify|k_unsort" -s 4 -c 4 -o /tmp/prof_$tag $C > gpurun_out/ncu_$tag.log 2>&1
  python tools/summarize_ncu.py /tmp/prof_$tag.ncu-rep > gpurun_out/r02_ncu_$tag.json
  python tools/ncu_hotlines.py /tmp/prof_$tag.ncu-rep "k_eval" 25 > gpurun_out/r02_ncu_${tag}_hotlines.txt
done
python tools/run_horner.py 1048576 > gpurun_out/horner_final.json 2>&1
du -sh gpurun_out
