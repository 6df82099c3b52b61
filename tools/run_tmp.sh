AB_ROUNDS=1 bash tools/lib_ab.sh "base L2 L3" --mx 0 --sweep 0
