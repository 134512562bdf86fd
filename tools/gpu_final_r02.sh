#!/bin/bash
# Round-2 final evidence: bench lines (cfg3 default, cfg5, cfg5 fp32, reference arm), the launch list of the bench
# command, ncu --set full of every cfg3 kernel and of the fp32 / real evaluators, smoke.  Each ncu pass runs
# after the same command exited 0 without ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
$CMD > gpurun_out/f_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/f_launches_cfg3.csv $CMD > gpurun_out/f_ncu_launch.log 2>&1
C3="python tools/run_cfg.py --config 3 --steps 1"
$C3 > gpurun_out/f_plain_c3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 9 -c 9 -o /tmp/prof_cfg3_f $C3 > gpurun_out/f_ncu_cfg3.log 2>&1
python tools/summarize_ncu.py /tmp/prof_cfg3_f.ncu-rep > gpurun_out/r02_ncu_cfg3_all_kernels.json
rm -f gpurun_out/r02_ncu_cfg3_hotlines.txt
for k in k_eval_tiled k_eval_mma k_classify_bucket k_bucket_hist k_unsort; do python tools/ncu_hotlines.py /tmp/prof_cfg3_f.ncu-rep $k 25 >> gpurun_out/r02_ncu_cfg3_hotlines.txt; done
for spec in "5:--fp32" "2:"; do
  cfg=${spec%%:*}; extra=${spec#*:}; tag=cfg${cfg}${extra:+_fp32}
  C="python tools/run_cfg.py --config $cfg $extra --steps 2"
  $C > gpurun_out/f_plain_$tag.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_classify|k_unsort|k_bucket_hist" -s 4 -c 4 -o /tmp/prof_$tag $C > gpurun_out/f_ncu_$tag.log 2>&1
  python tools/summarize_ncu.py /tmp/prof_$tag.ncu-rep > gpurun_out/r02_ncu_$tag.json
  python tools/ncu_hotlines.py /tmp/prof_$tag.ncu-rep "k_eval" 25 > gpurun_out/r02_ncu_${tag}_hotlines.txt
done
# the bench lines last, reading the traffic of the summary just captured
cp gpurun_out/r02_ncu_cfg3_all_kernels.json profiles/
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench_cfg3.json 2> gpurun_out/f_bench_cfg3.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_cfg5.json 2> gpurun_out/f_bench_cfg5.err
timeout 900 python bench.py --config 5 --fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_cfg5_fp32.json 2> gpurun_out/f_bench_cfg5_fp32.err
du -sh gpurun_out
