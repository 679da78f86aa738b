#!/bin/bash
# full GPU test suite + cfg4 / cfg1 step times + per-kind serialized profile
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
tag=${1:-w}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
tail -4 gpurun_out/${tag}_pytest.log
tools/tall_bench 1026 4 32 4 > gpurun_out/${tag}_tall.txt 2>&1; tail -2 gpurun_out/${tag}_tall.txt
timeout 600 python tools/step_time.py --config 4 --energies 4 --reps 2 > gpurun_out/${tag}_step4.txt 2>&1; cat gpurun_out/${tag}_step4.txt
timeout 600 python tools/step_time.py --config 1 --energies 16 --reps 5 > gpurun_out/${tag}_step1.txt 2>&1; cat gpurun_out/${tag}_step1.txt
timeout 600 python tools/group_kinds.py --config 4 --energies 4 --out gpurun_out/${tag}_gk4.json > gpurun_out/${tag}_gk4.txt 2>&1; head -3 gpurun_out/${tag}_gk4.txt
timeout 600 python tools/group_kinds.py --config 1 --energies 16 --out gpurun_out/${tag}_gk1.json > gpurun_out/${tag}_gk1.txt 2>&1; head -3 gpurun_out/${tag}_gk1.txt
