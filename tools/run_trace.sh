python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for c in 1 2 3; do python tools/trace_solve.py $c 3 --blocks > gpurun_out/t_$c.log 2>&1; head -1 gpurun_out/t_$c.log; grep median gpurun_out/t_$c.log; done
python tools/bench_frontier.py 5 2>&1 | tail -1
python tools/bench_windows.py 2000 0 2>&1 | tail -2
