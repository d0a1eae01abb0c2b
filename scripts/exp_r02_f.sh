# r02 experiment F: container loads for isolated 16-B rows + seams-first order (host fabs)
set -u
mkdir -p gpurun_out
{
echo "== ring_check"; timeout 600 python scripts/ring_check.py; echo "rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x -k "pinned or host or e2e or ring" 2>&1 | tail -3
} > gpurun_out/expF_check.txt 2>&1
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 5 "$@" 2>>gpurun_out/expF.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run C3 "" --config C3
run C3 "" --config C3
run C2 "" --config C2
run C4 "" --config C4
run C1 "" --config C1
} > gpurun_out/expF.txt 2>&1
cat gpurun_out/expF_check.txt gpurun_out/expF.txt
