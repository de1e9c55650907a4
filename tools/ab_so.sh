#!/bin/bash
# A/B two builds of the library on one box: ab_so.sh <a.so> <b.so> <command...>
set -u
A=$1; B=$2; shift 2
cp paper_2502_03000_b200/_lib/liblm_b200.so /tmp/cur.so
for r in 1 2; do
  for so in $A $B; do
    cp $so paper_2502_03000_b200/_lib/liblm_b200.so
    echo "== $so"; "$@"
  done
done
cp /tmp/cur.so paper_2502_03000_b200/_lib/liblm_b200.so
