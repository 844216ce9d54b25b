"""Debug: pscwin_dist_forward on a one-rank communicator, step by step (python tools/debug_nccl.py CASE)."""
import faulthandler, os, sys
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
faulthandler.dump_traceback_later(60, exit=True)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch, synth, oracle
import paper_2407_02109_b200 as pl
from paper_2407_02109_b200.bands import DistLayer, NcclComm
from gpu_util import BF16_TOL, dev, dev_weights, host, rel_err
i = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = [synth.tiny(H=32, W=16), synth.tiny(H=32, W=16, cycle_scan=1, mlp_hidden=128), synth.vitb(64, cycle_scan=1)][i]
x, w = synth.make_input(cfg), synth.make_weights(cfg)
dw = dev_weights(w, cfg)
desc = pl.LayerDesc.from_config(cfg)
xd = dev(x)
whole = pl.PSCWinLayer(desc, dw)(xd)
print("whole ok", flush=True)
comm = NcclComm(0, 1)
layer = DistLayer(desc, dw, 0, cfg.H, comm)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
xin = xd[0].contiguous()
with torch.cuda.stream(s):
    got = layer(xin)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
print("eager ok", rel_err(host(got), host(whole[0])), flush=True)
print("oracle", rel_err(host(got)[None], oracle.pscwin_layer(x, w, cfg)), flush=True)
out = torch.empty_like(got)
g = torch.cuda.CUDAGraph()
print("capturing", flush=True)
with torch.cuda.graph(g):
    layer(xin, out=out)
print("captured", flush=True)
out.zero_()
g.replay()
torch.cuda.synchronize()
print("replayed", torch.equal(out, got), flush=True)
comm.close()
print("ok")
