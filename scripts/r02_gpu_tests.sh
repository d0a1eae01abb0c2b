#!/bin/bash
# GPU test suite + smoke (round 2)
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -X faulthandler -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -c 2500 gpurun_out/gputest.log; tail -5 gpurun_out/smoke.log
