# compute-sanitizer over every device path (tools/sanitize_paths.py); one
# summary per tool under gpurun_out/san/ (copied to profiles/ as sanitizer_r02.txt).
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_paths.py \
        > gpurun_out/san/$tool.log 2>&1
    echo "== $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.log | tail -1)"
    grep -c MISMATCH gpurun_out/san/$tool.log
done
