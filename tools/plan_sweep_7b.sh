#!/bin/bash
for P in "auto:0,auto:0,auto:0,auto:0" "cluster:2,auto:0,auto:0,auto:0" "cluster:2,cluster:4,auto:0,auto:0" "auto:0,cluster:4,auto:0,auto:0" "auto:0,streamk:0,auto:0,auto:0" "auto:0,auto:0,cluster:2,auto:0" "auto:0,auto:0,auto:0,cluster:4" "cluster:2,auto:0,cluster:2,cluster:4"; do
  timeout 120 python tools/pf_bench.py --model 7b --depths=65536 --rounds 5 --plans $P 2>&1 | tail -1
done
