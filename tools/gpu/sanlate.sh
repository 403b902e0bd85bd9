# compute-sanitizer on the sanitizer workload incl. the late-wait in-step K1 (balanced and cost-model plans)
mkdir -p gpurun_out/san
timeout 600 python tools/sanitize_case.py > gpurun_out/san/plain.txt 2>&1; echo "plain rc=$?"
for t in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $t python tools/sanitize_case.py > gpurun_out/san/$t.txt 2>&1; echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$t.txt | head -1)"; done
