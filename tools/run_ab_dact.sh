set -u
out=gpurun_out/ab_dact; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mx.py -q -x > $out/parity.log 2>&1; tail -1 $out/parity.log
AB_ROUNDS=3 bash tools/lib_ab.sh "base direct direct6" --mx 0 --sweep 0
for f in gpurun_out/ab/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
    print(sys.argv[1].split('/')[-1], round(d['ms_per_step'],2), 'dA', round(k['gemm_dact_epilogue'],3), 'clk', d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
