# r02 experiment I: tile-ring ghost-only seam writes (w16 variant) vs whole sectors
set -u
mkdir -p gpurun_out
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 7 "$@" 2>>gpurun_out/expI.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
GHX_LIB=build/variants/w16.so GHX_RING=1 timeout 600 python scripts/ring_check.py | tail -2
for i in 1 2; do
run C3 "" --config C3
run C3 "GHX_LIB=build/variants/w16.so" --config C3
done
run C3x "" --config C3 --ngrow 2,0,0
run C3x "GHX_LIB=build/variants/w16.so" --config C3 --ngrow 2,0,0
run C2 "" --config C2
run C2 "GHX_LIB=build/variants/w16.so" --config C2
} > gpurun_out/expI.txt 2>&1
cat gpurun_out/expI.txt
