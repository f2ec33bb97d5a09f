#!/bin/bash
# run passbench with alternative builds of libqsim.so (tools/variants/*.so)
for v in tools/variants/*.so; do
  cp paper_2104_03293_b200/libqsim.so /tmp/libqsim_orig.so
  cp "$v" paper_2104_03293_b200/libqsim.so
  echo "== $v"; timeout 100 python tools/passbench.py --n 30 --reps 3
  cp /tmp/libqsim_orig.so paper_2104_03293_b200/libqsim.so
done
