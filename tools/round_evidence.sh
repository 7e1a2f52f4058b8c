# Round-end evidence: bench line, ncu launch list, one full ncu capture of
# k_solve (cfg 2), solve timelines.  Outputs under gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q > gpurun_out/ev/gpu_tests.log 2>&1; tail -1 gpurun_out/ev/gpu_tests.log
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err || tail -5 gpurun_out/ev/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
for c in 1 2 3; do python tools/trace_solve.py $c 3 --blocks > gpurun_out/ev/trace_cfg$c.txt 2>&1; done
python tools/probe_events.py 2 > gpurun_out/ev/probe_cfg2.txt 2>&1
python tools/probe_events.py 3 > gpurun_out/ev/probe_cfg3.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/ev/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve -c 1 -f \
    -o gpurun_out/ev/k_solve_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/ev/ncu_full.log 2>&1
tail -2 gpurun_out/ev/ncu_full.log
python tools/bench_frontier.py 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_frontier_f -c 1 -f \
    -o gpurun_out/ev/k_frontier_cfg3 python tools/bench_frontier.py 1 > gpurun_out/ev/ncu_frontier.log 2>&1
