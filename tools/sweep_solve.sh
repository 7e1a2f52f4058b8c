# Solve (cfg 1-3) and window-sequence (cfg 4) times of libevd variants (build_var/).
for lib in build_var/*.so; do
  echo "== $(basename $lib)"
  EVD_LIB=$lib python tools/time_solve.py ${CFGS:-1 2 3}
  EVD_LIB=$lib python tools/bench_windows.py 2000 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 windows/s', round(d['windows_per_s']), d['all_ok'])"
done
