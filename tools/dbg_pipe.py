import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
from tests.test_gpu_parity import _pipelined_launch_results, _shared_stream_grid
from tests import oracle_py as O
specs = _shared_stream_grid()
want = O.Oracle("reference").run_grid(specs, (0.5, 0.99))
ref_arr = np.concatenate([want["placement_hash"].view(np.float64), want["tail"].ravel(), want["total"].astype(np.float64)])
outs = _pipelined_launch_results()
n = len(specs)
for k, o in enumerate(outs):
    h = o[:n].view(np.uint64) != ref_arr[:n].view(np.uint64)
    t = o[n:3*n].view(np.uint64) != ref_arr[n:3*n].view(np.uint64)
    c = o[3*n:] != ref_arr[3*n:]
    print(os.environ.get("MSV_PIPELINE"), k, "hash bad", int(h.sum()), "tail bad", int(t.sum()), "total bad", int(c.sum()), np.nonzero(h)[0][:10])
