#!/bin/bash
mkdir -p gpurun_out
P=${TAG:-r02bb}
timeout 900 python tools/c4_stream_chunks.py 2 4 8 16 > gpurun_out/${P}_chunks.jsonl 2> gpurun_out/${P}_chunks.err; echo "rc=$?" >> gpurun_out/${P}_chunks.err
