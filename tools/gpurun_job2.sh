#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc $?"
timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag.json 2>&1; echo "diag rc $?"
timeout 300 python -m paper_1712_05878_b200.diag --batch 100 > gpurun_out/diag_b100.json 2>&1; echo "diag100 rc $?"
cat gpurun_out/diag.json
tail -3 gpurun_out/pytest_gpu2.log
