# full GPU suite + compute-sanitizer over tools/sanitize_small.py (racecheck also
# with the in-kernel F16S split off: its converter-group handoff goes through the
# tensor core's commit-arrive, which racecheck does not model)
exec > gpurun_out/stream_check.log 2>&1
timeout 1200 python -m pytest -q -x -m gpu tests/ 2>&1 | tail -2
echo "== memcheck"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py 2>&1 | tail -2
echo "== synccheck"; timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py 2>&1 | tail -2
echo "== racecheck"; timeout 900 compute-sanitizer --tool racecheck --print-limit 1 python tools/sanitize_small.py 2>&1 | grep -E "Error|SUMMARY|ok" | head -4
echo "== racecheck, in-kernel F16S split off"; MTNN_F16S_INKERNEL=0 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_small.py 2>&1 | tail -2
