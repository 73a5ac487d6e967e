# compute-sanitizer memcheck / racecheck / synccheck on small shapes of every engine
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.txt 2>&1; echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
cat gpurun_out/sanitize_rc.txt; for tool in memcheck racecheck synccheck; do echo "== $tool"; tail -8 gpurun_out/sanitize_$tool.txt; done
