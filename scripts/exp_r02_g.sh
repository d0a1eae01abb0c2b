# r02 experiment G: host e2e, default build vs container-load variant (build/variants/cont.so)
set -u
mkdir -p gpurun_out
run() {  # label envs args...
  local label=$1 envs=$2; shift 2
  r=$(env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-split --e2e-steps 5 "$@" 2>>gpurun_out/expG.err)
  echo "$label [$envs $*] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(e["value"], e["ms_per_step"], e["verified"])' 2>&1 | tail -1)"
}
{
run C3 "" --config C3
run C3 "GHX_LIB=build/variants/cont.so" --config C3
run C3 "" --config C3
run C3 "GHX_LIB=build/variants/cont.so" --config C3
run C2 "" --config C2
run C2 "GHX_LIB=build/variants/cont.so" --config C2
run C3 "GHX_RING_TILE=0" --config C3
} > gpurun_out/expG.txt 2>&1
cat gpurun_out/expG.txt
