# r02 experiment E: host-memory task order with tile ring tasks
set -u
mkdir -p gpurun_out
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 5 "$@" 2>>gpurun_out/expE.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run C3 "" --config C3
run C3 "GHX_NO_INTERLEAVE=1" --config C3
run C3 "GHX_BULK_FIRST=1" --config C3
run C3yz "" --config C3 --ngrow 0,2,2
run C3 "GHX_HOST_BLOCKS=6" --config C3
run C3 "GHX_HOST_BLOCKS=12" --config C3
run C3 "" --config C3
run C2 "GHX_NO_INTERLEAVE=1" --config C2
run C2 "GHX_BULK_FIRST=1" --config C2
} > gpurun_out/expE.txt 2>&1
cat gpurun_out/expE.txt
