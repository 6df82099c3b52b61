#!/usr/bin/env bash
# The round's measurement suite in one GPU call (run from the repo root on the B200 box):
#   gpurun --timeout 3000 -- 'bash tools/measure_round.sh v13'
# then, here:   python tools/ncu_traffic.py gpurun_out/v13/full_raw.csv > profiles/rNN_ncu_traffic.json
#               python tools/ncu_summary.py launches gpurun_out/v13/launches.csv > profiles/rNN_ncu_launches_v13.md
#               python tools/ncu_summary.py full gpurun_out/v13/full_raw.csv > profiles/rNN_ncu_full_v13_c1.md
set -u
tag=${1:-latest}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi --query-gpu=name,serial,clocks.max.sm,power.limit --format=csv,noheader > "$out/box.txt"
python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1
python -m pytest tests -m gpu -q > "$out/gputests.log" 2>&1
# the headline line (Mixtral layer, EP = 1, tuner's C; per-C sweep, MXFP8 variants, cpu_baseline)
python bench.py > "$out/bench.json" 2> "$out/bench.err"
# the other BASELINE configs on one GPU
for c in "mixtral 8" "dsv3 8" "qwen3 8" "qwen3 1"; do
  set -- $c
  python bench.py --config "$1" --ep-emulate "$2" --sweep 1 --no-cpu-baseline > "$out/cfg_$1_ep$2.json" 2>&1
done
python bench.py --config qwen3 --placement contiguous --sweep 0 --mx 0 --no-cpu-baseline > "$out/cfg_qwen3_contig_ep1.json" 2>&1
# config 5 and the MACT-over-training comparison (Methods 1-3)
timeout 900 python tools/budget_sweep.py > "$out/budget_sweep.json" 2> "$out/budget_sweep.err"
timeout 1200 python tools/mact_over_training.py > "$out/mact.json" 2> "$out/mact.err"
# energy per FLOP at the power cap (cuBLAS vs the layer, sustained) and per-clock GEMM efficiency
timeout 600 python tools/sustained_clock.py > "$out/sustained.json" 2> "$out/sustained.err"
timeout 600 python tools/gemm_vs_cublas.py > "$out/gemm_vs_cublas.json" 2> "$out/gemm_vs_cublas.err"
timeout 300 python tools/router_bench.py > "$out/router.json" 2> "$out/router.err"
# ncu: launch list of the bench command, then one full capture (DRAM bytes per launch)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches.csv" \
  python bench.py --steps 2 --warmup 1 --mx 0 --sweep 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"gemm_kernel|dispatch_scatter|gather_reduce" -c 11 -o "$out/full" \
  python bench.py --steps 1 --warmup 0 --mx 0 --sweep 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i "$out/full.ncu-rep" --page raw --csv > "$out/full_raw.csv" 2>/dev/null
tail -1 "$out/gputests.log"
tail -1 "$out/smoke.log"
