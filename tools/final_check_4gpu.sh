python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_4.log 2>&1; tail -3 gpurun_out/pytest_gpu_4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29912 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29913 bench.py --gpus 4 --config 3 --steps 3 --no-e2e > gpurun_out/bench_n4_cfg3.json 2> gpurun_out/bench_n4_cfg3.err
for f in bench_n2 bench_n4 bench_n4_cfg3; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step'],2), (d.get('e2e') or {}).get('value'), d.get('imbalance'), d['clocks']['sm_mhz'])"; done
