# the flat-grid columnwise MX quantiser vs the previous build (git stash of csrc/mx.cu + kernels.h):
# bench.py's mxfp8_wgrad variant, mx_quant_colwise kernel class, interleaved
mkdir -p gpurun_out/mxq
timeout 600 python -m pytest tests/test_gpu_mx.py tests/test_gpu_pdl.py -q -x > gpurun_out/mxq/tests.log 2>&1; tail -1 gpurun_out/mxq/tests.log
for r in 1 2; do for b in new old; do
  if [ $b = old ]; then cp paper_2511_21431_b200/libmemfine_old.so paper_2511_21431_b200/libmemfine.so.ab; else cp paper_2511_21431_b200/libmemfine_new.so paper_2511_21431_b200/libmemfine.so.ab; fi
  cp paper_2511_21431_b200/libmemfine.so.ab paper_2511_21431_b200/libmemfine.so
  timeout 400 python bench.py --sweep 0 --no-cpu-baseline > gpurun_out/mxq/b_${b}_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/mxq/b_${b}_$r.json').read().strip().splitlines()[-1]);v=d['variants']['mxfp8_wgrad']
print('$b', round(d['ms_per_step'],2), round(v['ms_per_step'],2), round(v['kernel_ms_per_step']['mx_quant_colwise'],3), d['clocks']['sm_mhz'])"
done; done
cp paper_2511_21431_b200/libmemfine_new.so paper_2511_21431_b200/libmemfine.so
