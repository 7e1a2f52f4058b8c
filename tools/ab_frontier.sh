# Same-box A/B of the cfg-3 frontier for build_var/{base,new}.so (twice, interleaved)
mkdir -p gpurun_out/ab
for r in 1 2; do for v in ${AB_VARS:-base new}; do [ -f build_var/$v.so ] || continue; echo "== $v"; EVD_LIB=build_var/$v.so timeout 300 python tools/bench_frontier.py 5 tiles 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['seconds_per_call'], d['median_s'], d['marks'], d['checksum'])"; done; done > gpurun_out/ab/frontier.log 2>&1
cat gpurun_out/ab/frontier.log
