# Source-level ncu capture of the solve's event pass at a narrow node
# (evd_probe_events, cfg 2, width 1e-4: the 5th probe launch):
# gpurun_out/probe_narrow.ncu-rep
timeout 600 ncu --section SourceCounters --section WarpStateStats --section InstructionStats \
   --import-source on --clock-control none -k regex:k_event_probe --launch-skip 4 -c 1 \
   -o gpurun_out/probe_narrow -f python tools/probe_events.py 2 3 > gpurun_out/probe_narrow.log 2>&1
