# r02 experiment L: phased host exchange as three launches (faces on a wider grid)
set -u
mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests/test_gpu_random.py tests/test_gpu_parity.py -q -x -m gpu -k "random or phased or pinned" 2>&1 | tail -2
} > gpurun_out/expL_check.txt 2>&1
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 7 "$@" 2>>gpurun_out/expL.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run C3 "GHX_PHASE_LAUNCHES=0" --config C3
run C3 "" --config C3
run C3 "GHX_HOST_FACE_BLOCKS=16" --config C3
run C3 "GHX_HOST_FACE_BLOCKS=64" --config C3
run C3 "GHX_HOST_FACE_BLOCKS=148" --config C3
run C2 "GHX_PHASE_LAUNCHES=0" --config C2
run C2 "" --config C2
run C4 "GHX_PHASE_LAUNCHES=0" --config C4
run C4 "" --config C4
} > gpurun_out/expL.txt 2>&1
cat gpurun_out/expL_check.txt gpurun_out/expL.txt
