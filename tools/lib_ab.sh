# A/B of several builds of libmemfine.so on ONE box, interleaved: each ab_libs/<name>.so (git-ignored, but it
# travels to the box with the snapshot - gpurun_out/ does not) is copied over the in-tree library and the bench
# runs with the given arguments; two rounds.  The in-tree library is restored at the end.
#   bash tools/lib_ab.sh "base S X" --mx 0 --sweep 0        -> gpurun_out/ab/<name>_<round>.json
set -eu
names=$1; shift
out=gpurun_out/ab; mkdir -p $out
lib=paper_2511_21431_b200/libmemfine.so
cp $lib $out/.intree.so
for n in $names; do [ -f ab_libs/$n.so ] || { echo "missing ab_libs/$n.so" >&2; exit 1; }; done
for i in $(seq 1 ${AB_ROUNDS:-2}); do
  for n in $names; do
    cp ab_libs/$n.so $lib
    timeout 900 python bench.py --no-cpu-baseline "$@" > $out/${n}_$i.json 2> $out/${n}_$i.err || true
  done
done
cp $out/.intree.so $lib
