# evd_probe_events timings of libevd variants (built into build_var/).
for lib in build_var/*.so; do
  for c in ${CFGS:-2 3}; do
    echo "$(basename $lib) $(EVD_LIB=$lib python tools/probe_events.py $c 2>&1 | tail -1)"
  done
done
