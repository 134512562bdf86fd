mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/run_precondition.py > gpurun_out/precond.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "precondition or partial or cover or analyse or smoke or newton" > gpurun_out/precond_tests.log 2>&1; echo "rc=$?" >> gpurun_out/precond_tests.log
