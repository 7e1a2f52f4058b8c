mkdir -p gpurun_out/ab
python -m pytest tests -m gpu -q -x > gpurun_out/ab/gpu_tests.log 2>&1; tail -2 gpurun_out/ab/gpu_tests.log
for r in 1 2; do for v in base new; do echo "== $v"; EVD_LIB=build_var/$v.so python tools/time_solve.py 1 2 3; done; done > gpurun_out/ab/time.log 2>&1
for v in base new; do echo "== $v"; EVD_LIB=build_var/$v.so python tools/bench_frontier.py 3 2>&1 | tail -2; done > gpurun_out/ab/frontier.log 2>&1
python bench.py --no-cpu > gpurun_out/ab/bench.json 2> gpurun_out/ab/bench.err
cat gpurun_out/ab/time.log gpurun_out/ab/frontier.log
