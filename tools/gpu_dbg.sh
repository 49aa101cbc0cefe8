#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/host_overhead.py pinned > gpurun_out/ho_pinned.json 2>&1
timeout 300 python tools/host_overhead.py upload > gpurun_out/ho_upload.json 2>&1
SSJB_STREAM=0 timeout 300 python tools/host_overhead.py upload > gpurun_out/ho_upload_nostream.json 2>&1
SSJB_LIB=$PWD/paper_1711_07295_b200/lib/libssjoin_head.so timeout 300 python tools/host_overhead.py upload > gpurun_out/ho_upload_head.json 2>&1
SSJB_LIB=$PWD/paper_1711_07295_b200/lib/libssjoin_head.so timeout 300 python tools/host_overhead.py pinned > gpurun_out/ho_pinned_head.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:rescan_saturated -c 1 -o gpurun_out/rescan python tools/c2_phases.py 128 1 > gpurun_out/ncu_rescan.log 2>&1
