# GPU session script (edited per call)
mkdir -p gpurun_out
( echo "# compute-sanitizer on tools/sanitize_cases.py (APT_TABLE=none; one small launch of every kernel family, each checked vs the oracle), one B200"
for tool in memcheck synccheck racecheck; do echo "## $tool"; APT_TABLE=none timeout 900 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | grep -v "^\[" | tail -40; echo "rc=$?"; done ) > gpurun_out/r2_compute_sanitizer.txt 2>&1
grep -E "^##|ERROR SUMMARY|RACECHECK SUMMARY|Error" gpurun_out/r2_compute_sanitizer.txt | head -30
timeout 900 python -m pytest tests -m gpu -x -q -k "repack or pf_ or mxf4_matches or prefill_full" 2>&1 | tail -2
