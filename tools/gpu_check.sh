#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + full capture.
# usage (from this container): gpurun --timeout 1800 -- 'bash tools/gpu_check.sh [tag]'
tag=${1:-r01}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi_$tag.txt 2>&1
python -m paper_2511_12376_b200._build > gpurun_out/build_$tag.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
if [ "${NCU:-1}" = 1 ]; then
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:delta_(encode_ws|decode_tma|offsets)' -c 3 -f -o gpurun_out/prof_$tag $CMD \
    > gpurun_out/ncu_full_$tag.log 2>&1
fi
echo done
