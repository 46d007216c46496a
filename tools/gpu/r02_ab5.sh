for rep in 1 2; do for v in default prev; do
  lib=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; [ $v = prev ] && lib=$PWD/build/variants/prev/libmtnn_b200.so
  MTNN_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v sweep',round(d['value'],1),d['clocks']['sm_mhz'])"
done; done
