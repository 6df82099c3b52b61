# MEMFINE_FLAG_WGRAD_OVERLAP: parity test, then per-C steps with and without it (same box, interleaved)
set -u
out=gpurun_out/wov; mkdir -p $out; rm -f $out/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wgrad_overlap or chunking_invariance" > $out/test.log 2>&1; tail -3 $out/test.log
for i in 1 2; do
  for c in ${WOV_CFGS:-"mixtral 1"}; do
    set -- $c
    for f in 0 1; do
      timeout 600 python bench.py --config $1 --ep-emulate $2 --mx 0 --sweep 1 --no-cpu-baseline --wgrad-overlap $f > $out/${1}_ep$2_f${f}_$i.json 2> $out/${1}_ep$2_f${f}_$i.err
      python -c "
import json,sys
try:
    d=json.loads(open('$out/${1}_ep$2_f${f}_$i.json').read().strip().splitlines()[-1])
    print('$1 ep$2 wov=$f r$i', {c:round(v.get('ms_per_step',0),2) for c,v in d['per_C'].items()}, 'clk', d['clocks']['sm_mhz'])
except Exception as e: print('$1 $f ERR', e); print(open('$out/${1}_ep$2_f${f}_$i.err').read()[-1500:])
"
    done
  done
done
for f in 0 1; do
  timeout 600 python bench.py --mx 0 --sweep 0 --chunks 8 --no-cpu-baseline --wgrad-overlap $f > $out/c8_f$f.json 2>&1
  python -c "
import json
d=json.loads(open('$out/c8_f$f.json').read().strip().splitlines()[-1]); print('C=8 wov=$f', round(d['ms_per_step'],2), {a:round(b,2) for a,b in d['kernel_ms_per_step'].items()})"
done
