#!/bin/bash
# Quick GPU iteration: gpu tests (subset or all), timeline of config B, bench A/B.
TAG=${TAG:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu ${TESTS:-tests} > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -3 gpurun_out/${TAG}_pytest.txt
timeout 300 python tools/timeline.py B 7 > gpurun_out/${TAG}_timeline.txt 2>/dev/null; head -3 gpurun_out/${TAG}_timeline.txt | tail -1
VARIANTS="${VARIANTS:-base}" bash tools/ab.sh
