#!/bin/bash
# One iteration: build, stage times of cfg3 / cfg4 / cfg5 / cfg5-fp32 / cfg2, then the GPU suite.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
rm -f gpurun_out/iter_times.txt
for spec in "3:" "3:" "4:" "2:" "5:" "5:--fp32"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/iter_times.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/iter_tests.log 2>&1; echo "rc=$?" >> gpurun_out/iter_tests.log
