OUT=gpurun_out; mkdir -p $OUT
: > $OUT/sanitizer_r2n.txt
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $OUT/sanitizer_r2n.txt
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > $OUT/san_$tool.log 2>&1; echo "exit $?" >> $OUT/sanitizer_r2n.txt
  grep -E "ERROR SUMMARY|sanitize run complete|Error|ok$" $OUT/san_$tool.log | tail -8 >> $OUT/sanitizer_r2n.txt
done
echo done
