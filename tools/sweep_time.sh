# evd_solve device time of libevd variants (built into build_var/).
for lib in build_var/*.so; do
  echo "$(basename $lib)"; EVD_LIB=$lib python tools/time_solve.py ${CFGS:-1 2 3}
done
