#!/bin/bash
# L2 bulk prefetch distance of the Σ sandwich producer (QT_SAND_PF): per-kernel times on the profiling slice, FP64 and FP32.
cp paper_1912_10024_b200/libqtsse.so /tmp/libqtsse.cur.so
for v in cur sandpf4 sandpf8 sandpf16 sandpf32; do
  [ "$v" != cur ] && cp variants/$v.so paper_1912_10024_b200/libqtsse.so
  echo "== $v"; python tools/kt.py prof; python tools/kt.py prof fp32
  cp /tmp/libqtsse.cur.so paper_1912_10024_b200/libqtsse.so
done
