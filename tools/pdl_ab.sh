mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pdl/gputests.log 2>&1; tail -1 gpurun_out/pdl/gputests.log
for r in 1 2 3; do for v in 1 0; do
  MEMFINE_PDL=$v timeout 300 python bench.py --sweep 0 --mx 0 --no-cpu-baseline > gpurun_out/pdl/b_${v}_$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pdl/b_${v}_$r.json').read().strip().splitlines()[-1]);print('pdl=$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(sum(d['kernel_ms_per_step'].values()),3))"
done; done
