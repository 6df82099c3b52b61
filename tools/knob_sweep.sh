#!/usr/bin/env bash
# Per-kernel in-step times of the headline workload under the GEMM launch knobs (one box, back to back):
#   gpurun -- 'bash tools/knob_sweep.sh TAG'   ->  gpurun_out/TAG/knobs.jsonl
set -u
tag=${1:-knobs}
out=gpurun_out/$tag
mkdir -p "$out"
run() {
  local name=$1; shift
  env "$@" python bench.py --steps 8 --warmup 3 --sweep 0 --mx 0 --no-cpu-baseline 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'knob': '$name', 'ms': d['ms_per_step'], 'e2e_ms': d['e2e']['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz'], 'k': d['kernel_ms_per_step']}))" >> "$out/knobs.jsonl"
}
run base
run l2_8 MEMFINE_L2_GROUP_MB=8
run l2_48 MEMFINE_L2_GROUP_MB=48
run l2_96 MEMFINE_L2_GROUP_MB=96
run cta1 MEMFINE_GEMM_CTA=1
run wave MEMFINE_WAVE_SYNC=1
run base2
cat "$out/knobs.jsonl"
