out=gpurun_out/kb; mkdir -p $out
for c in "qwen3 8 1" "qwen3 8 2" "mixtral 8 1" "mixtral 8 4" "qwen3 8 1" "qwen3 8 2"; do
  set -- $c
  python bench.py --config $1 --ep-emulate $2 --chunks $3 --mx 0 --sweep 0 --no-cpu-baseline > $out/$1_$2_$3.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$out/$1_$2_$3.json').read().strip().splitlines()[-1]); print('$1 ep$2 C=$3', round(d['ms_per_step'],2), {a[:14]:round(b,3) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
