for rep in 1 2; do for f in 0 64 32; do timeout 200 python tools/quick_bench.py --cfg 5 --variant uniform_1e-2 --reps 6 --flags $f 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print('flags', $f, round(r['tflops']), [round(x) for x in r['exec_ms']], r['class_tflops'][2])"; done; done
