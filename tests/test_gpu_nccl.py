"""The real NCCL path of the group-sharded engine (csrc/sps.cu `gather`, ncclAllGather on the context
stream): G = 2 ranks under torchrun against G = 1 and the oracle (groups never
exchange particles; only the per-step statistics are gathered).  Needs >= 2 GPUs; skipped otherwise
(this build's GPU pool gives one -- the sharded engine is then covered by the loopback transport,
tests/test_gpu_multirank.py)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import paper_1304_4333_b200 as sps, sps_synth
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
ids = [sps.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(ids, src=0)
X, y = sps_synth.config_data("cfg2", n=300)
cov = sps.g_prior(X, 2, 1.0 / 16, device=rank)
ctx = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=1, rank=rank, nranks=world, nccl_id=ids[0], device=rank)
r = ctx.run()
ctx.close()
if rank == 0:
    print("RESULT" + json.dumps(dict(L=r["L"], t=[int(v) for v in r["t_cycle"]], R=[int(v) for v in r["R_cycle"]],
                                     logml=r["logml"], nse=r["logml_nse"], mean=list(r["mean"]))))
dist.destroy_process_group()
"""


@pytest.mark.gpu
def test_nccl_two_ranks_match_one_rank_and_oracle(orc, tmp_path):
    import numpy as np
    import torch

    import sps_synth

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one per rank)")
    import paper_1304_4333_b200 as sps

    sps.build()
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = orc.g_prior(X, 2, 1.0 / 16)
    o = orc.run(X, y, 2, 8, 256, seed=1, prior_mean=np.zeros(25), prior_cov=cov)
    script = tmp_path / "child.py"
    script.write_text(CHILD.format(root=ROOT))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    g = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")][-1][6:])
    assert g["L"] == o["L"] and g["t"] == list(o["t_cycle"]) and g["R"] == list(o["R_cycle"])
    assert abs(g["logml"] - o["logml"]) <= 1e-6 and abs(g["nse"] - o["logml_nse"]) <= 1e-6
    assert np.all(np.abs(np.array(g["mean"]) - o["mean"]) <= 1e-6)


@pytest.mark.gpu
def test_nccl_transport_one_rank_exchange_path(orc, tmp_path):
    """The exchange code path of the sharded engine -- stats slices, ESS partials, group (m, s) and L_j
    all-gathered by ncclAllGather on the context stream, the finalize as its own launch, host-driven M
    steps -- over a real one-rank NCCL communicator (SPS_XCHG_1RANK=1; include/sps.h).  On a 1-GPU pool
    this is the only execution of the NCCL transport: launched exactly like the 2-rank test (torchrun,
    torch.distributed nccl, the id broadcast), against the oracle with the same bars."""
    import numpy as np
    import torch

    import sps_synth

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1304_4333_b200 as sps

    sps.build()
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = orc.g_prior(X, 2, 1.0 / 16)
    o = orc.run(X, y, 2, 8, 256, seed=1, prior_mean=np.zeros(25), prior_cov=cov)
    script = tmp_path / "child.py"
    script.write_text(CHILD.format(root=ROOT))
    env = dict(os.environ, SPS_XCHG_1RANK="1", NCCL_DEBUG="WARN")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", "29534", str(script)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    g = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")][-1][6:])
    assert g["L"] == o["L"] and g["t"] == list(o["t_cycle"]) and g["R"] == list(o["R_cycle"])
    assert abs(g["logml"] - o["logml"]) <= 1e-6 and abs(g["nse"] - o["logml_nse"]) <= 1e-6
    assert np.all(np.abs(np.array(g["mean"]) - o["mean"]) <= 1e-6)
    # the same run on the default one-rank path (no exchange): identical schedule
    s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=1)
    r = s.run()
    s.close()
    assert r["L"] == g["L"] and list(r["R_cycle"]) == g["R"] and abs(r["logml"] - g["logml"]) <= 1e-9
