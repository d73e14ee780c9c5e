#!/bin/bash
# mixed-mode timing for the in-tree library and tools/variants/*.so
L=paper_2407_12208_b200/libmpkmeans.so
cp $L /tmp/lib_base.so
for v in /tmp/lib_base.so tools/variants/*.so; do
  cp $v $L
  echo "== $(basename $v)"
  python tools/mixed_time.py c3_blobs_1m_d64 2.0 5
  python tools/mixed_time.py c5_vq_10m 2.0 1
  MPK_MIXED_SMALL=1 python tools/mixed_time.py c3_blobs_1m_d64 2.0 5
done
cp /tmp/lib_base.so $L
