# ncu --set full of one cfg-5 solve (k_solve_spec<768>, 5.3 M events):
# gpurun_out/ev/k_solve_cfg5.ncu-rep
mkdir -p gpurun_out/ev
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_solve_spec -c 1 -f \
    -o gpurun_out/ev/k_solve_cfg5 python tools/time_solve.py 5 > gpurun_out/ev/ncu_cfg5.log 2>&1
