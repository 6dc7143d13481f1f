#!/bin/bash
# resident quantizer: parity (resident on), C2 timing, stage timing build
tag=${1:-x}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -m paper_2511_12376_b200._build > /dev/null 2>&1
export BSNP_RESIDENT=1
timeout 120 python tools/lab_resident.py > gpurun_out/labr_$tag.log 2>&1
timeout 900 python -m pytest tests/test_quantizer_gpu.py tests/test_store_gpu.py -x -q >> gpurun_out/labr_$tag.log 2>&1
if [ "${RT:-1}" = 1 ]; then
python -c "from paper_2511_12376_b200 import _build; _build.build(force=True, extra=['-DBSNP_RTIMING'])" > /dev/null 2>&1
timeout 120 python tools/lab_resident.py >> gpurun_out/labr_$tag.log 2>&1
python -m paper_2511_12376_b200._build --force > /dev/null 2>&1
fi
if [ "${NCU:-0}" = 1 ]; then
LOG2N=28 timeout 120 python tools/lab_resident.py > gpurun_out/plain_res_$tag.log 2>&1 && LOG2N=28 timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_resident -s 2 -c 1 -f -o gpurun_out/prof_res_$tag python tools/lab_resident.py > gpurun_out/ncu_res_$tag.log 2>&1
fi
