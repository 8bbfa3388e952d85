#!/bin/bash
# Row-stream prototype (scripts/proto/): bit-exactness and timings vs the product SpMV.
mkdir -p gpurun_out
(cd scripts/proto && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC -o libstream_proto.so stream_proto.cu)
timeout 900 python scripts/proto/run_proto.py ${PROTO_SPECS:-C3:2048:1024 C3:2048:4096 C2:2048:1024 C4:2048:1024} > gpurun_out/r02_proto.jsonl 2> gpurun_out/r02_proto.err
echo "rc=$?"; cat gpurun_out/r02_proto.jsonl; tail -5 gpurun_out/r02_proto.err
