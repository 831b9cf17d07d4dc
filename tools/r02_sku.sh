#!/bin/bash
# Σ sandwich k-loop unroll (QT_SAND_KU) on the profiling slice, FP64 and FP32 (experiment; default stays 2).
cp paper_1912_10024_b200/libqtsse.so /tmp/cur.so
for v in cur sku1 sku5 sku10; do
  [ "$v" != cur ] && cp variants/$v.so paper_1912_10024_b200/libqtsse.so
  echo "== $v"; python tools/kt.py prof; python tools/kt.py prof fp32
  cp /tmp/cur.so paper_1912_10024_b200/libqtsse.so
done
