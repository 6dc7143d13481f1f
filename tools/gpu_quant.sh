#!/bin/bash
# Quantizer timings (C2) + ncu launch list and full capture of the quant kernels.
tag=${1:-q01}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2511_12376_b200._build > gpurun_out/build_$tag.log 2>&1
timeout 600 python tools/lab_quant.py > gpurun_out/labq_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/labq_$tag.log
BSNP_FUSED=1 timeout 600 python tools/lab_quant.py > gpurun_out/labq_fused_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/labq_fused_$tag.log
BSNP_FUSED=1 timeout 900 python -m pytest tests -m gpu -x -q -k fused > gpurun_out/pytest_fused_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused_$tag.log
if [ "${NCU:-1}" = 1 ]; then
CMD="python tools/lab_quant.py"
export LOG2N=30
timeout 300 $CMD > gpurun_out/plainq_$tag.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launchesq_$tag.csv $CMD > gpurun_out/ncuq_launch_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:(fit_|quantize_kernel|dequantize_kernel)' -c 6 -f -o gpurun_out/profq_$tag $CMD \
    > gpurun_out/ncuq_full_$tag.log 2>&1
fi
echo done
