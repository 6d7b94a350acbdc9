"""Small runs of every kernel path for compute-sanitizer (memcheck /
racecheck / synccheck): stencil (one lane per row), 27-pt (4 lanes/row),
power-law through the CSR-stream kernel (its auto choice) and through the
row-block kernel (all classes) + warp-per-row, 3 LOCAL ranks (pack,
exchange, unpack, combine), fp32, per-destination schedules;
round 2: the TMA-fed CSR-stream kernel, aliased sends, the explicit END
combine, LOCAL group graphs (copy and put, device-resident epoch), and the
pipelined apply_host (streamed-x instantiation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
from paper_2203_02530_b200 import dspmv as D
from oracle import schedules as S
from tests.gpu_helpers import LocalRun, derive_ops, oracle_ops_to_lib

V, E, _ = S.fine_dag([-1, 1])
FINE = oracle_ops_to_lib(S.derive(S.topological_orders(E, V)[5], {v: i % 2 for i, v in enumerate(V)}))

cases = [("7pt", 16 ** 3, gen.stencil("7pt", (16, 16, 16)), D.DSPMV_SKERNEL_AUTO),
         ("27pt", 12 ** 3, gen.stencil("27pt", (12, 12, 12)), D.DSPMV_SKERNEL_AUTO),
         ("pl", 6000, gen.powerlaw(6000), D.DSPMV_SKERNEL_AUTO),
         ("pl-block", 6000, gen.powerlaw(6000), D.DSPMV_SKERNEL_BLOCK),
         ("pl-tma", 6000, gen.powerlaw(6000), D.DSPMV_SKERNEL_STREAM_TMA)]
for name, n, (rp, col, val), sk in cases:
    for P in (1, 3):
        for dt in (D.DSPMV_F64, D.DSPMV_F32):
            for ex in (D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT):
                v = val.astype(np.float32) if dt == D.DSPMV_F32 else val
                for gran, ops in (("coarse", derive_ops()), ("fine", FINE)):
                    if gran == "fine" and name.startswith("pl"):
                        continue                      # power-law: every rank is a peer, offsets +-1, +-2
                    run = LocalRun(n, rp, col, v, P, dtype=dt, exchange=ex, s_kernel=sk)
                    y = run.apply(run.schedule(ops), gen.x_values((0, n)), reps=2)
                    run.close()
                    assert np.isfinite(y).all()
                    print(name, P, dt, ex, gran, "ok", flush=True)
import torch  # noqa: E402
stream = torch.cuda.Stream()
n = 16 ** 3
rp, col, val = gen.stencil("27pt", (16, 16, 16))
for ex in (D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT):
    for opts in ({"pack_mode": D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS}, {"accumulate_mode": D.DSPMV_ACC_EXPLICIT_IN_END}):
        run = LocalRun(n, rp, col, val, 3, exchange=ex, **opts)
        ss = run.schedule(derive_ops())
        xs, ys = run.xy(gen.x_values((0, n)))
        D.dspmv_apply_group(ss, xs, ys)
        for _ in range(2):
            D.dspmv_apply_graph_group(ss, xs, ys, stream)
        torch.cuda.synchronize()
        assert all(bool(torch.isfinite(y).all()) for y in ys)
        run.close()
        print("group graph", ex, opts, "ok", flush=True)
# pipelined apply_host (x streamed in chunks: the coherent-load instantiation)
n = 64 ** 3
rp, col, val = gen.stencil("7pt", (64, 64, 64))
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
sch = D.dspmv_schedule_create(plan, derive_ops(), 2)
xh = torch.from_numpy(gen.x_values((0, n))).pin_memory()
yh = torch.empty_like(xh).pin_memory()
for _ in range(2):
    D.dspmv_apply_host(sch, xh, yh)
assert bool(torch.isfinite(yh).all())
D.dspmv_schedule_destroy(sch)
D.dspmv_plan_destroy(plan)
D.dspmv_comm_destroy(comm)
print("apply_host pipeline ok", flush=True)
D.dspmv_l2_flush(0)
print("sanitize run complete")
