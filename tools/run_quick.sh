python tools/diag_spill.py c2 0 2>&1 | tail -9 | grep -v hdr | grep -v examples
timeout 600 python bench.py --steps 3 --warmup 2 --views-per-rank 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); print('FPS', round(d['value'],1)); print({k: round(v['ms_per_view'],3) for k,v in d['stages'].items()}); print(d['counters_per_view'])"
