#!/bin/bash
cp paper_2101_07344_b200/liblatecache_b200.so /tmp/libcur.so
for L in C; do
  cp bisect_libs/lib$L.so paper_2101_07344_b200/liblatecache_b200.so
  echo "== $L"; timeout 300 python -m pytest tests/test_gpu_parity.py -q  2>&1 | tail -3
done
cp /tmp/libcur.so paper_2101_07344_b200/liblatecache_b200.so
