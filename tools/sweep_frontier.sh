# cfg-3 frontier time of libevd variants (built into build_var/).
for lib in build_var/*.so; do
  echo "$(basename $lib) $(EVD_LIB=$lib python tools/bench_frontier.py 1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['seconds_per_call']*1e3, 2), 'ms', d['marks'])")"
done
