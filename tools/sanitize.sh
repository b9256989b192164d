#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the kernel parity tests and one C1
# executor pass (smoke). Logs to gpurun_out/sanitize_*.log; summary lines to stdout.
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="flash_attention or gemm_majors or layernorm or softmax_xent or bias_grad_and_adam or gemm_splitk"
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_kernels_gpu.py -q -x -k "$SEL" > gpurun_out/sanitize_${tool}_kernels.log 2>&1
  echo "$tool kernels rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_${tool}_kernels.log | tail -2 | tr '\n' ' ')"
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$? $(grep -E 'ERROR SUMMARY|smoke' gpurun_out/sanitize_${tool}_smoke.log | tail -2 | tr '\n' ' ')"
done
