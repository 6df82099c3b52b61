# A/B of wave pacing settings on one box: bench.py --mx 0 --sweep 0, interleaved repeats
out=gpurun_out/$1; mkdir -p $out
nvidia-smi --query-gpu=serial,clocks.max.sm --format=csv,noheader > $out/box.txt
for rep in 1 2 3; do for cfg in "off 0 1" "s1 -1 1" "s2 -1 2" "s4 -1 4"; do set -- $cfg
  MEMFINE_WAVE_SYNC=$2 MEMFINE_PACE_SLACK=$3 python bench.py --mx 0 --sweep 0 --no-cpu-baseline > $out/mix_$1_$rep.json 2>&1
  MEMFINE_WAVE_SYNC=$2 MEMFINE_PACE_SLACK=$3 python bench.py --config dsv3 --ep-emulate 8 --mx 0 --sweep 0 --no-cpu-baseline > $out/dsv3_$1_$rep.json 2>&1
done; done
