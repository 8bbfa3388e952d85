#!/bin/bash
# compute-sanitizer evidence (memcheck / racecheck / synccheck / initcheck) for the
# SpMV kernels and the converter, on small C2-like (27-pt stencil) and C3-like
# (power-law with heavy groups) inputs, the fp32 handle, the host pipelines, the
# fused multi-GPU peer step (virtual ranks) and the 2-process CUDA IPC peer step.
# Summaries land in gpurun_out/sanitize_<tool>.txt.
mkdir -p gpurun_out
SEL_PARITY='test_stencil27 or (test_powerlaw_heavy_groups and 128-1) or test_fp32_handle or test_spmv_groups_writes_only_its_rows or test_host_async_stream or test_host_staged_pipeline or test_e8 or test_empty_rows or test_all_zero'
SEL_PEER='test_spmv_peer_stores or (test_peer_power_iteration_virtual_ranks and 2) or test_spmv_norm2_fused or test_interior_boundary_split'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 --target-processes all \
      python -m pytest tests/test_gpu_parity.py tests/test_peer.py tests/test_multigpu_device.py -q -x -p no:cacheprovider \
      -k "$SEL_PARITY or $SEL_PEER" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.txt | tail -4
done
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 \
    python -m pytest tests/test_peer.py -q -x -p no:cacheprovider -k "two_processes_ipc" > gpurun_out/sanitize_memcheck_ipc.txt 2>&1
echo "ipc memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_memcheck_ipc.txt | tail -4
