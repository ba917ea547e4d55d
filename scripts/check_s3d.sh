#!/bin/bash
# session-3 check: cull/list tests, smem action-bitmap A/B, rev diagnostics
mkdir -p gpurun_out/s3d
timeout 900 python -m pytest tests/test_gpu_mapops.py tests/test_gpu_refpipeline.py tests/test_gpu_api.py tests/test_gpu_steady.py -q -m gpu -x > gpurun_out/s3d/pytest.log 2>&1; tail -2 gpurun_out/s3d/pytest.log
REPS=3 STAGES="fuse_rev" bash scripts/abenv2.sh "" "LM_REV_ABITS=0" 2>&1 | tee gpurun_out/s3d/ab_abits.txt
LM_B200_LIB=$PWD/ab/diag.so timeout 300 python tools/diag_apply.py > gpurun_out/s3d/diag.txt 2>&1; cat gpurun_out/s3d/diag.txt
