# compute-sanitizer racecheck / synccheck on one small double-hoisted forward (tools/sanitize_forward.py)
for tool in racecheck synccheck; do
  SAN_B=17 timeout 900 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_forward.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
done
