import sys, struct, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2105_07829_b200 as bpc
from workloads import *
w = Config("dbg", "custom", Comp(SCALED_SIGN, use_ef=1), numels=(300000,), threshold_bytes=0)
import os
if os.environ.get("KIND") == "ld": w = Config("dbg", "custom", Comp(LINEAR_DITHER, bits=7, use_ef=0), numels=(300000,), threshold_bytes=0)
offs, D = layout(w.tensor_numels())
ctx = bpc.context_for(w, rank=0, world_size=1)
x = torch.tensor(gen_params(w), device="cuda")
ocfg = oracle.Cfg.from_workload(w, n=1); ost = oracle.State(1, D, gen_params(w))
g = gen_grad(w, 0, 1)
delta, p, gt = oracle.round_(ocfg, ost, g[None], 1e-3)
ctx.compress(torch.tensor(g, device="cuda")); ctx.aggregate(); ctx.step(x, 1e-3); ctx.sync()
send = ctx.copy_state(bpc.BUF_SEND); pb = ctx.copy_state(bpc.BUF_P)
etl = np.frombuffer(ctx.copy_state(bpc.BUF_SERVER_ERR).tobytes(), np.float32)
for ci, (po, nb) in enumerate(ocfg.payload_layout()):
    c = ctx.chunk(ci)
    gs = struct.unpack('<f', send[c.payload_offset:c.payload_offset+4].tobytes())[0]
    os_ = struct.unpack('<f', delta[0, po:po+4].tobytes())[0]
    gp = struct.unpack('<f', pb[c.payload_offset:c.payload_offset+4].tobytes())[0]
    op = struct.unpack('<f', p[po:po+4].tobytes())[0]
    print(ci, c.len, 'worker s gpu/orc', gs, os_, 'server s gpu/orc', gp, op, 'ratio', gp/op)
    e_g = etl[c.server_err_offset:c.server_err_offset+c.len]; e_o = ost.et[c.offset:c.offset+c.len]
    print('   etl gpu[:4]', e_g[:4], 'orc', e_o[:4], 'ndiff', np.count_nonzero(e_g != e_o))
    dg = oracle.decompress(ocfg.s.comp, pb[c.payload_offset:c.payload_offset+nb].tobytes(), c.len)
    Dg = e_g + dg
    print('   Delta gpu unique |.|', np.unique(np.abs(Dg))[:5], 'L1/L', np.sum(np.abs(Dg.astype(np.float64)))/c.len)
