# Solve timelines of libevd variants (built into build_var/) on configs 2 and 3.
for lib in build_var/*.so; do
  for c in ${CFGS:-2 3}; do
    EVD_LIB=$lib EVD_SOLVE_FILTER=0 python tools/trace_solve.py $c 3 > /tmp/t.log 2>&1
    echo "$(basename $lib) $(head -1 /tmp/t.log)"; grep median /tmp/t.log
  done
done
