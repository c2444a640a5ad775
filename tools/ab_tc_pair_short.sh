for rep in 1 2; do for f in 0 32; do for c in 3 4; do timeout 200 python tools/quick_bench.py --cfg $c --size 32768 --reps 5 --flags $f 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print('cfg', $c, 'flags', $f, round(r['tflops']), [round(x,1) for x in r['exec_ms']], r['class_tflops'])"; done; done; done
