# Source-level ncu capture of one event pass (evd_probe_events, cfg 2, w = 1)
# for build_var/$1.so: gpurun_out/probe_src_$1.ncu-rep
v=${1:-base}
EVD_LIB=build_var/$v.so timeout 600 ncu --section SourceCounters --section WarpStateStats --section InstructionStats \
   --import-source on --clock-control none -k regex:k_event_probe -c 1 -o gpurun_out/probe_src_$v -f \
   python tools/probe_events.py 2 2 > gpurun_out/probe_src_$v.log 2>&1
