import sys, json, torch
sys.path.insert(0, '.')
import bench, numpy as np
import paper_2403_12179_b200 as amr
from paper_2403_12179_b200 import comm, _native as N
for name in ("C3", "C2"):
    cfg = bench.scaled(bench.CONFIGS[name], 1)
    L = bench.layout(amr, cfg, 1)
    mf, _ = bench.make_fields(amr, cfg, L)
    plan = comm.plan_build_fill_boundary(mf, L["geom"])
    rows = mf.storage_rows()
    st = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
    out = {}
    for tag, flag in (("all", 0), ("xfaces", N.EXEC_ONLY_XFACES), ("rest", N.EXEC_NO_XFACES), ("yzfaces", 0x800)):
        ex = comm.Executor(plan, 0, N.EXEC_DIRECT | flag, rows, mf.ncomp, rows, mf.ncomp, 0, 0, mf.ncomp, 8, 0)
        b = ex.bind(comm._table(ex, mf, [(mf.local_indices, mf._ptrs)]), st.cuda_stream)
        for _ in range(3): b.run(st.cuda_stream)
        ts = []
        for _ in range(20):
            flush.zero_(); torch.sum(clean)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); b.run(st.cuda_stream); e1.record(st); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        out[tag] = (round(sum(ts) / len(ts), 4), ex.ntags)
    print(name, json.dumps(out), flush=True)
    del mf
    torch.cuda.empty_cache()
