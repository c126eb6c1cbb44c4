#!/bin/bash
mkdir -p gpurun_out
export LPQT_LIB=build/variants/lib_trace.so
timeout 120 python tools/chain_trace.py --graph > gpurun_out/chain.log 2>&1
timeout 120 python tools/chain_trace.py --graph --shapes 4096x11008 > gpurun_out/chain_down.log 2>&1
head -6 gpurun_out/chain.log; grep -A7 "4096, 11008" gpurun_out/chain.log; cat gpurun_out/chain_down.log
