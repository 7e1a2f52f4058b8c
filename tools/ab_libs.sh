# Same-box A/B of two libevd builds: build_var/base.so and build_var/new.so
# (e.g. the working tree built with a -D switch off and on).  GPU tests on the
# working tree, then cfg 1-3 solve times and the cfg-3 frontier for each
# library (EVD_LIB), twice, interleaved.  Outputs under gpurun_out/ab/.
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab/gpu_tests.log 2>&1; tail -2 gpurun_out/ab/gpu_tests.log
for r in 1 2; do for v in base new; do echo "== $v"; EVD_LIB=build_var/$v.so timeout 300 python tools/time_solve.py 1 2 3; done; done > gpurun_out/ab/time.log 2>&1
for v in base new; do echo "== $v"; EVD_LIB=build_var/$v.so timeout 300 python tools/bench_frontier.py 3 2>&1 | tail -1 | cut -c1-200; done > gpurun_out/ab/frontier.log 2>&1
cat gpurun_out/ab/time.log gpurun_out/ab/frontier.log
