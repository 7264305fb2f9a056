"""The one-process-per-GPU path under torchrun (NCCL): par_eliminate with
transport="process" and bench.py's multi-rank loop.  gpurun gives one GPU, so
these run at nproc=1 (the broadcast/gather code paths execute; the world-size
2/3 logic is covered by tests/test_dist_gloo.py on CPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import torch, torch.distributed as dist
dist.init_process_group("nccl")
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
from _util import build_input, load_golden
from golden.digest import digest_parts
from paper_1308_1536_b200 import MatrixBuffer, Precision, par_eliminate, ZeroPivot
from paper_1308_1536_b200.scalars import canonical_bits
meta, arrays = load_golden({name!r})
A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), build_input(meta, arrays))
try:
    trace, minors, stats = par_eliminate(A, dist.get_world_size(), transport="process",
                                         collect_minors=meta["collect_minors"], series=meta["series"])
except ZeroPivot as exc:
    trace, minors = exc.trace, exc.series
rows = []
if minors is not None:
    for m in minors.sizes():
        r = minors.rows[m]
        rows.append((m, [canonical_bits(x) for x in r.signed],
                     None if r.normalized is None else [canonical_bits(x) for x in r.normalized]))
dig = digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series], rows,
                   [canonical_bits(x) for row in A.rows for x in row])
if dist.get_rank() == 0:
    open({out!r}, "w").write(dig)
dist.destroy_process_group()
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["uniform13_s5_p192", "zero_pivot3", "uniform24_s2_p4096"])
def test_torchrun_process_transport(name, tmp_path):
    from _util import load_golden
    meta, _ = load_golden(name)
    script = tmp_path / "run.py"
    out = tmp_path / "digest.txt"
    script.write_text(SCRIPT.format(root=ROOT, name=name, out=str(out)))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                    "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script)],
                   check=True, timeout=600, cwd=ROOT)
    assert out.read_text() == meta["digest"]


def test_bench_under_torchrun_small():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
                        "--steps", "1", "--warmup", "1", "--dim", "96", "--bits", "512", "--family", "random",
                        "--cpu-seconds", "1", "--dist"], timeout=600, cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0


SCRIPT_LA = r'''
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("nccl")
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.parexec import dist_run
from paper_1308_1536_b200.synth import random_uniform_soa
n, p = {n}, {p}
A = random_uniform_soa(n, p, seed=41)
eng = DeviceElimination(n, p, "real", local, dist.get_rank(), dist.get_world_size())
eng.load(A)
_, pbytes = eng.pivot_buffer()
pivot = torch.empty(pbytes, dtype=torch.uint8, device=f"cuda:{{local}}")
eng.lib.ds_use_pivot_buffer(eng.ctx, pivot.data_ptr(), pbytes)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.lib.ds_set_stream(eng.ctx, stream.cuda_stream)
failed = dist_run(eng, n, True, True, pivot, lambda t, src: dist.broadcast(t, src=src))
res = HostResults.alloc(n, 1, eng.L, True)
eng.results(n, res)
fin = A.copy()
eng.fetch(fin)
np.savez({out!r}, limbs=fin.limbs, exp=fin.exp, cls=fin.cls, dl=res.dets.limbs, de=res.dets.exp,
         sl=res.signed.limbs, se=res.signed.exp, sc=res.signed.cls, flags=res.row_flags)
eng.close()
dist.destroy_process_group()
'''


def test_torchrun_lookahead_matches_single_process(tmp_path):
    """The caller-driven lookahead (dist_run: tile split, next-pivot exchange on the
    lookahead stream, multipliers there) gives the single-process engine's results."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from paper_1308_1536_b200.engine import DeviceElimination, HostResults
    from paper_1308_1536_b200.synth import random_uniform_soa
    n, p = 300, 1024
    script = tmp_path / "la.py"
    out = tmp_path / "la.npz"
    script.write_text(SCRIPT_LA.format(root=ROOT, n=n, p=p, out=str(out)))
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                    "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script)],
                   check=True, timeout=600, cwd=ROOT)
    z = np.load(out)
    A = random_uniform_soa(n, p, seed=41)
    with DeviceElimination(n, p, "real") as eng:
        eng.load(A)
        res = HostResults.alloc(n, 1, eng.L, True)
        eng.run(True, True, 0, n, res)
        fin = A.copy()
        eng.fetch(fin)
    assert np.array_equal(z["limbs"], fin.limbs) and np.array_equal(z["exp"], fin.exp)
    assert np.array_equal(z["cls"], fin.cls)
    assert np.array_equal(z["dl"], res.dets.limbs) and np.array_equal(z["de"], res.dets.exp)
    assert np.array_equal(z["flags"], res.row_flags)
    for m in range(2, n + 1):
        sl = slice((m - 1) * n, (m - 1) * n + m)
        assert np.array_equal(z["sl"][:, :, sl], res.signed.limbs[:, :, sl])
        assert np.array_equal(z["se"][:, sl], res.signed.exp[:, sl])


def test_bench_two_ranks_one_gpu_gloo():
    """bench.py's multi-rank loop (row-cyclic shards, per-step pivot broadcast, max-over-ranks
    timing) with 2 ranks on this box's one GPU: gloo with host staging stands in for NCCL (two
    ranks may not share a device under NCCL).  The rank-0 JSON line reports n_gpus = 2 and the
    parity leg is skipped (it needs the whole matrix on one rank)."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                        "--steps", "1", "--warmup", "1", "--dim", "160", "--bits", "1024", "--family", "random",
                        "--no-cpu", "--dist-backend", "gloo"], timeout=900, cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0


def test_bench_power_family_small():
    """bench.py on the complex Artless power family (leading N x N block of genmat.power_matrix), with
    the parity leg checking the run against the oracle."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "1", "--dim", "64", "--bits", "1024",
                        "--family", "power", "--cpu-seconds", "1", "--parity-m", "32"], timeout=900, cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["config"]["kind"] == "complex" and d["parity"]["ok"], d["parity"]
