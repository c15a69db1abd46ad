cd /root/repo
run() { echo "== $*"; env A=1 timeout 200 python bench.py --config $1 --steps 20 --warmup 3 --no-cpu-baseline 2>/tmp/err | tail -1 > /tmp/o.json; python -c "
import json; d=json.loads(open('/tmp/o.json').read()); print(round(d['value'],1), 'Gpts/s', round(d['ms_per_step'],4), 'ms', {k: round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, 'alg1', d.get('alg1') and round(d['alg1']['value'],1))" || tail -3 /tmp/err; }
run c4
run c2
run c4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
