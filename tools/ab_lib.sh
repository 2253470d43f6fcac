#!/bin/bash
# Dev A/B of two builds of the library on one box: alternates ab_old.so / ab_new.so (repo root)
# under the same probe command, REPS times each; the in-tree library is restored to ab_new.so.
# Usage: REPS=2 bash tools/ab_lib.sh "<command>" > log
LIB=paper_1805_04590_b200/libdts_b200.so
for r in $(seq 1 ${REPS:-2}); do
  for v in old new; do
    cp ab_$v.so $LIB
    echo "== $v $r"
    eval "$1"
  done
done
cp ab_new.so $LIB
