#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bk}
timeout 1200 python tools/prefix_phases.py c4 --bitmap f3 > gpurun_out/${P}_c4_prefix.jsonl 2> gpurun_out/${P}_c4_prefix.err; echo "rc=$?" >> gpurun_out/${P}_c4_prefix.err
