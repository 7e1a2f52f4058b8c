# Solve times at forced CTA sizes (EVD_SOLVE_BLOCK) with build_var/new.so
mkdir -p gpurun_out/ab
for r in 1 2; do for b in default 640 768 512; do echo "== $b"; if [ $b = default ]; then EVD_LIB=build_var/new.so timeout 300 python tools/time_solve.py ${CFGS:-2 3 5}; else EVD_SOLVE_BLOCK=$b EVD_LIB=build_var/new.so timeout 300 python tools/time_solve.py ${CFGS:-2 3 5}; fi; done; done > gpurun_out/ab/threads.log 2>&1
cat gpurun_out/ab/threads.log
