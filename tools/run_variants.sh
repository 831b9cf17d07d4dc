#!/bin/bash
# usage (on the GPU box): tools/run_variants.sh <config> v1 v2 ...  — per-kernel times of each variants/<v>.so
cfg=$1; shift
cp paper_1912_10024_b200/libqtsse.so /tmp/libqtsse.cur.so
for v in "$@"; do
  cp variants/$v.so paper_1912_10024_b200/libqtsse.so
  echo "== $v"; python tools/kt.py $cfg
done
cp /tmp/libqtsse.cur.so paper_1912_10024_b200/libqtsse.so
