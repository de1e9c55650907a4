#!/bin/bash
# A/B several builds of the library on one box: ab_multi.sh "<a.so> <b.so> ..." <command...>
set -u
LIBS=$1; shift
cp paper_2502_03000_b200/_lib/liblm_b200.so /tmp/cur.so
for r in 1 2; do
  for so in $LIBS; do
    cp $so paper_2502_03000_b200/_lib/liblm_b200.so
    echo "== $so"; "$@"
  done
done
cp /tmp/cur.so paper_2502_03000_b200/_lib/liblm_b200.so
