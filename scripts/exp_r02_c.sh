# r02 experiment C: e2e (pinned host fabs over PCIe) on C3 -- direction split and host grid
set -u
mkdir -p gpurun_out
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --e2e-steps 5 "$@" 2>>gpurun_out/expC.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run all ""
run x "" --ngrow 2,0,0
run yz "" --ngrow 0,2,2
run all "GHX_HOST_BLOCKS=4"
run all "GHX_HOST_BLOCKS=16"
run all "GHX_HOST_BLOCKS=32"
run all "GHX_RING=0"
run x "GHX_HOST_BLOCKS=16" --ngrow 2,0,0
run yz "GHX_HOST_BLOCKS=16" --ngrow 0,2,2
run yz "GHX_HOST_BLOCKS=32" --ngrow 0,2,2
} > gpurun_out/expC.txt 2>&1
cat gpurun_out/expC.txt
