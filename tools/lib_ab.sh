# A/B two builds of libmemfine.so on one box: the in-tree build (new) against $1 (base), interleaved runs of
# the bench (extra bench args after the first argument).
set -u
base=$1; shift
out=gpurun_out/ab; mkdir -p $out
cp paper_2511_21431_b200/libmemfine.so $out/libmemfine_new.so
for i in 1 2; do
  for v in new base; do
    cp $out/libmemfine_$v.so paper_2511_21431_b200/libmemfine.so
    [ $v = base ] && cp $base paper_2511_21431_b200/libmemfine.so
    timeout 900 python bench.py --no-cpu-baseline "$@" > $out/${v}_$i.json 2> $out/${v}_$i.err
  done
done
cp $out/libmemfine_new.so paper_2511_21431_b200/libmemfine.so
