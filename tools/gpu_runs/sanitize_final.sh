# compute-sanitizer over every kernel family at the end of round 2
mkdir -p gpurun_out/sanf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sanf/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  for fam in map slices rows skinny coop scan stream; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_check.py $fam > gpurun_out/sanf/${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanf/${tool}_${fam}.log | tail -1)" >> gpurun_out/sanf/summary.txt
  done
done
