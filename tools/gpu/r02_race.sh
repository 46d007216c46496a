exec > gpurun_out/race.log 2>&1
echo "== HEAD"; timeout 600 compute-sanitizer --tool racecheck --print-limit 1 python tools/probes/race_one.py 128 2048 256 2>&1 | grep -E "SUMMARY|ok"
echo "== HEAD in-kernel off"; timeout 600 compute-sanitizer --tool racecheck --print-limit 1 python -c "
import sys; sys.path.insert(0,'.')
from paper_1702_03192_b200 import _lib
_lib.config_set('f16s_inkernel_max_short', 0)
sys.argv=['x','128','2048','256']; exec(open('tools/probes/race_one.py').read())" 2>&1 | grep -E "SUMMARY|ok|Error"
echo "== 305cd74"; MTNN_B200_LIB=build/wt305/paper_1702_03192_b200/lib/libmtnn_b200.so timeout 600 compute-sanitizer --tool racecheck --print-limit 1 python tools/probes/race_one.py 128 2048 256 2>&1 | grep -E "SUMMARY|ok"
echo "== 305cd74 sanitize_small"; MTNN_B200_LIB=build/wt305/paper_1702_03192_b200/lib/libmtnn_b200.so timeout 900 compute-sanitizer --tool racecheck --print-limit 1 python tools/sanitize_small.py 2>&1 | grep -E "SUMMARY|ok"
