# Same-box A/B/C of up to three libevd builds (build_var/{pre,base,new}.so,
# whichever exist): cfg 1-3 solve times, twice, interleaved.
mkdir -p gpurun_out/ab
for r in 1 2; do for v in ${AB_VARS:-pre base new}; do [ -f build_var/$v.so ] || continue; echo "== $v"; EVD_LIB=build_var/$v.so timeout 300 python tools/time_solve.py 1 2 3; done; done > gpurun_out/ab/time.log 2>&1
cat gpurun_out/ab/time.log
