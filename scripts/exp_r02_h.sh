# r02 experiment H: phased host exchange -- parity (golden / random / pinned) and e2e
set -u
mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests/test_gpu_random.py tests/test_gpu_parity.py -q -x -m gpu -k "random or phased or pinned" 2>&1 | tail -4
echo "== ring_check"; timeout 600 python scripts/ring_check.py | tail -3
echo "== ring_check phased"; GHX_PHASED=1 timeout 600 python scripts/ring_check.py | tail -3
} > gpurun_out/expH_check.txt 2>&1
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 5 "$@" 2>>gpurun_out/expH.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"], e.get("exec"))' 2>&1 | tail -1)"
}
{
run C3 "" --config C3
run C3 "GHX_PHASED=0" --config C3
run C3 "" --config C3
run C2 "" --config C2
run C2 "GHX_PHASED=0" --config C2
run C4 "" --config C4
run C1 "" --config C1
run C5 "" --config C5
} > gpurun_out/expH.txt 2>&1
cat gpurun_out/expH_check.txt gpurun_out/expH.txt
