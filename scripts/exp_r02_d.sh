# r02 experiment D: tile ring tasks (host-memory x seams): correctness + C3/C2 e2e
set -u
mkdir -p gpurun_out
{
echo "== ring_check tile"; timeout 600 python scripts/ring_check.py; echo "rc=$?"
echo "== ring_check column (GHX_RING_TILE=0)"; GHX_RING_TILE=0 timeout 600 python scripts/ring_check.py; echo "rc=$?"
} > gpurun_out/expD_check.txt 2>&1
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 5 "$@" 2>>gpurun_out/expD.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run C3 "" --config C3
run C3x "" --config C3 --ngrow 2,0,0
run C3 "GHX_RING_TILE=0" --config C3
run C3x "GHX_RING_TILE=0" --config C3 --ngrow 2,0,0
run C3x "GHX_HOST_BLOCKS=16" --config C3 --ngrow 2,0,0
run C3x "GHX_HOST_BLOCKS=4" --config C3 --ngrow 2,0,0
run C2 "" --config C2
run C2 "GHX_RING_TILE=0" --config C2
run C4 "" --config C4
run C4 "GHX_RING_TILE=0" --config C4
} > gpurun_out/expD.txt 2>&1
cat gpurun_out/expD_check.txt gpurun_out/expD.txt
