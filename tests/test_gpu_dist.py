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
