set -u
out=gpurun_out/r02d_val
mkdir -p $out
nvidia-smi --query-gpu=name,serial,clocks.max.sm,power.limit --format=csv,noheader > $out/box.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $out/gputests.log 2>&1
python bench.py > $out/bench.json 2> $out/bench.err
tail -1 $out/gputests.log; tail -1 $out/smoke.log; tail -c 600 $out/bench.json
