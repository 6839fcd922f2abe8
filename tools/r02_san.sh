O=gpurun_out/r02_san
mkdir -p $O
for tool in memcheck synccheck racecheck; do
  echo "## $tool" >> $O/san.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 8 python tools/sanitize_probe.py >> $O/san.txt 2>&1; echo "rc=$?" >> $O/san.txt
done
grep -E "^## |ERROR SUMMARY|RACECHECK SUMMARY|rc=|probe done" $O/san.txt
