# interleaved same-box A/B of runtime knobs over configs:
#   bash tools/env_ab.sh "dsv3:8 qwen3:1" "base:X=0 l2_8:MEMFINE_L2_GROUP_MB=8 ..."  -> gpurun_out/env_ab/<cfg>.jsonl
set -u
cfgs=$1; knobs=$2
out=gpurun_out/env_ab; mkdir -p $out
for i in $(seq 1 ${AB_ROUNDS:-2}); do
  for c in $cfgs; do
    cfg=${c%%:*}; ep=${c##*:}
    for kv in $knobs; do
      name=${kv%%:*}; envs=${kv#*:}
      env ${envs//,/ } timeout 600 python bench.py --config $cfg --ep-emulate $ep --steps 8 --warmup 3 --sweep 0 --mx 0 --no-cpu-baseline 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'knob': '$name', 'round': $i, 'ms': round(d['ms_per_step'],3), 'sm_mhz': d['clocks']['sm_mhz'], 'k': {a[5:]: round(b,3) for a,b in d['kernel_ms_per_step'].items() if a.startswith('gemm')}}))" >> $out/${cfg}_ep$ep.jsonl
    done
  done
done
for f in $out/*.jsonl; do echo "== $f"; cat $f; done
