# usage: bash tools/run_ab_generic.sh "<lib names>" "<pytest files>" [bench args...]
# parity tests on the in-tree build, then an interleaved same-box A/B of ab_libs/<name>.so builds
set -u
names=$1; tests=$2; shift 2
out=gpurun_out/ab_run; mkdir -p $out
rm -f gpurun_out/ab/*.json
if [ -n "$tests" ]; then timeout 1200 python -m pytest $tests -q -x > $out/parity.log 2>&1; tail -1 $out/parity.log; fi
AB_ROUNDS=${AB_ROUNDS:-3} bash tools/lib_ab.sh "$names" "$@"
for f in gpurun_out/ab/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
    print(sys.argv[1].split('/')[-1], round(d['ms_per_step'],2), ' '.join(f"{a[5:]}={b:.3f}" for a,b in k.items() if a.startswith('gemm')), 'clk', d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
