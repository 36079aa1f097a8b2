"""One launch of the NN gradients kernel at the bench config (for ncu)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2211_00621_b200 import _lib
npts, nin, nout = 1 << 20, 64, 16
dev = torch.device("cuda")
x = torch.randn(npts * nin, dtype=torch.float64, device=dev) * 0.5
y = torch.randint(0, nout, (npts,), dtype=torch.int32, device=dev)
w = torch.randn(nin * nout, dtype=torch.float64, device=dev) * 0.3
b = torch.randn(nout, dtype=torch.float64, device=dev) * 0.1
loss = torch.empty(1, dtype=torch.float64, device=dev)
dw = torch.empty(nin * nout, dtype=torch.float64, device=dev)
db = torch.empty(nout, dtype=torch.float64, device=dev)
err = torch.full((1,), -1, dtype=torch.int64, device=dev)
lib = _lib.load()
ws = torch.zeros(lib.pmx_nn_workspace_bytes(npts, nin, nout), dtype=torch.uint8, device=dev)
for _ in range(2):
    _lib.check(lib.pmx_nn_softmax_grad_f64(x.data_ptr(), y.data_ptr(), w.data_ptr(), b.data_ptr(), npts, nin, nout,
                                           loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(),
                                           err.data_ptr(), torch.cuda.current_stream().cuda_stream), "nn")
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "time":
    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        a.record()
        lib.pmx_nn_softmax_grad_f64(x.data_ptr(), y.data_ptr(), w.data_ptr(), b.data_ptr(), npts, nin, nout,
                                    loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(),
                                    err.data_ptr(), torch.cuda.current_stream().cuda_stream)
        bb.record()
        bb.synchronize()
        ts.append(a.elapsed_time(bb))
    print("nn ms min", min(ts), "med", sorted(ts)[10], "loss", float(loss.item()))
