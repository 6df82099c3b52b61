# same-box A/B of ab_libs builds over several configs: bash tools/run_ab_cfgs.sh "base new" "dsv3:8 qwen3:8 qwen3:1"
set -u
names=$1; cfgs=$2
res=gpurun_out/ab_cfgs; mkdir -p $res
for c in $cfgs; do
  cfg=${c%%:*}; ep=${c##*:}
  rm -f gpurun_out/ab/*.json
  AB_ROUNDS=${AB_ROUNDS:-3} bash tools/lib_ab.sh "$names" --config $cfg --ep-emulate $ep --mx 0 --sweep 0
  mkdir -p $res/${cfg}_ep$ep; cp gpurun_out/ab/*.json $res/${cfg}_ep$ep/
  for f in $res/${cfg}_ep$ep/*.json; do python - "$f" "$c" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
    print(sys.argv[2], sys.argv[1].split('/')[-1], round(d['ms_per_step'],2), ' '.join(f"{a[5:]}={b:.3f}" for a,b in k.items() if a.startswith('gemm')), 'clk', d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
  done
done
