#!/bin/bash
# usage (on the GPU box): tools/run_variants_cmd.sh "<command>" v1 v2 ... — run a command with each variants/<v>.so
cmd=$1; shift
cp paper_1912_10024_b200/libqtsse.so /tmp/libqtsse.cur.so
for v in "$@"; do
  cp variants/$v.so paper_1912_10024_b200/libqtsse.so
  echo "== $v"; bash -c "$cmd"
done
cp /tmp/libqtsse.cur.so paper_1912_10024_b200/libqtsse.so
