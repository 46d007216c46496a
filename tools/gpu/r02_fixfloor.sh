for rep in 1 2; do for v in default fixfloor nofix; do
  lib=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; fx=1
  [ $v = fixfloor ] && lib=$PWD/build/variants/fixfloor/libmtnn_b200.so
  [ $v = nofix ] && fx=0
  MTNN_FIXUP=$fx MTNN_B200_LIB=$lib timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v fcn',round(d['value'],1))"
  MTNN_FIXUP=$fx MTNN_B200_LIB=$lib timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v single',round(d['ms_per_step']*1e3,1),'us')"
done; done
