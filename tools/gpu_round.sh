#!/bin/bash
# Full GPU check: build, all GPU tests, smoke, bench (b200 + reference arm),
# ncu launch list of the bench's kernels and a full capture of the C1 and C2
# top kernels.  Outputs under gpurun_out/ with the given tag.
tag=${1:-r}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -m paper_2511_12376_b200._build > gpurun_out/build_$tag.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$tag.log
s=$(date +%s.%N)
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
rc=$?; echo "bench wall $(python -c "print(round($(date +%s.%N) - $s, 1))") s rc=$rc" >> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
if [ "${NCU:-1}" = 1 ]; then
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-c0 --no-ckpt --no-sweep"
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k "regex:delta_(encode_ws|decode_tma|count|scan)|fit_sum|fit_label|quantize_codes|dequantize_kernel" -c 8 -f -o gpurun_out/prof_$tag $CMD \
    > gpurun_out/ncu_full_$tag.log 2>&1
  # the cluster encode / dequantize kernels of one C2 encode + dequantize
  timeout 300 python tools/lab_quant_once.py > gpurun_out/plainq_$tag.log 2>&1 && \
  REPS=1 DEQ=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:fit_sum|fit_label|quantize_codes|dequantize_kernel" -c 4 -f -o gpurun_out/profq_$tag \
    python tools/lab_quant_once.py > gpurun_out/ncu_fullq_$tag.log 2>&1
fi
echo done
