# full GPU suite + compute-sanitizer over tools/sanitize_small.py (session-4 build, 4+5 in-kernel rings)
exec > gpurun_out/stream_check2.log 2>&1
timeout 1200 python -m pytest -q -x -m gpu tests/ 2>&1 | tail -2
echo "== memcheck"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py 2>&1 | tail -2
echo "== synccheck"; timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py 2>&1 | tail -2
echo "== racecheck"; timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_small.py 2>&1 | tail -2
