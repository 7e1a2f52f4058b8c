# Round-end evidence (run under gpurun from the repo root): GPU tests, the
# bench line (+ the reference arm), the fp64 / shared-atomic peaks, the ncu
# launch list of the bench command and one `ncu --set full` capture each of
# the solve kernel (cfg 2) and the tiled frontier kernel (cfg 3).
# Outputs under gpurun_out/ev/; tools/profiles_update.py copies the summaries
# into profiles/.
set -x
mkdir -p gpurun_out/ev
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bench_fp64 tools/bench_fp64.cu && \
    ./tools/bench_fp64 > gpurun_out/ev/fp64_peak.json
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/gpu_tests.log 2>&1; tail -1 gpurun_out/ev/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err || tail -5 gpurun_out/ev/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
for c in 1 2 3; do timeout 300 python tools/trace_solve.py $c 3 --blocks > gpurun_out/ev/trace_cfg$c.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/ev/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve -c 1 -f \
    -o gpurun_out/ev/k_solve_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu --no-extra \
    > gpurun_out/ev/ncu_full.log 2>&1
tail -2 gpurun_out/ev/ncu_full.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_frontier_tiles -c 1 -f \
    -o gpurun_out/ev/k_frontier_tiles_cfg3 python tools/bench_frontier.py 1 tiles > gpurun_out/ev/ncu_frontier.log 2>&1
tail -2 gpurun_out/ev/ncu_frontier.log
