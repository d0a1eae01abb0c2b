# r02 experiment B: bulk-row placement variants + public-call overhead
set -u
mkdir -p gpurun_out
{
VSTEPS=50 bash scripts/variants.sh C2 "GHX_BULK=0" "GHX_BULK=1"
VSTEPS=50 bash scripts/variants.sh C4 "GHX_BULK=0" "GHX_BULK=1"
VSTEPS=50 bash scripts/variants.sh C3 "GHX_BULK=1" "GHX_BULK=0" "GHX_BULK_FIRST=1" "GHX_NO_CHAIN=1"
VSTEPS=50 bash scripts/variants.sh C3 "GHX_BULK=1|--ngrow 2,0,0" "GHX_BULK=1|--ngrow 0,2,2" "GHX_BULK=0|--ngrow 0,2,2"
} > gpurun_out/expB_times.txt 2>&1
timeout 300 python scripts/call_overhead.py > gpurun_out/expB_overhead.txt 2>&1
cat gpurun_out/expB_times.txt; head -30 gpurun_out/expB_overhead.txt
