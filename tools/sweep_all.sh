# Solve / windows / frontier timings of libevd variants (built into build_var/).
for lib in build_var/*.so; do
  echo "== $(basename $lib)"
  EVD_LIB=$lib python tools/time_solve.py ${CFGS:-1 2 3}
  EVD_LIB=$lib python tools/bench_windows.py 2000 74 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 windows/s', round(d['windows_per_s']), d['all_ok'])"
  EVD_LIB=$lib python tools/bench_frontier.py 1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3 frontier ms', round(d['seconds_per_call']*1e3, 2), d['marks'])"
done
