"""The multi-GPU training path (TrainEngine.step with world_size > 1:
ugs_backward -> all-reduce of the AoS-12 gradient -> ugs_adam_step) run with
two ranks on the one available B200 over gloo (NCCL refuses two ranks on one
device).  Checks: the replicas stay bitwise identical (densify included), and
world=2 x batch=B matches one process with batch=2B (same global mean
gradient, different summation order)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from conftest import load_golden  # noqa: E402

ITERS, B = 12, 2


def _dataset():
    import paper_2505_05643_b200 as ug
    z = load_golden("train.npz")
    slices = [ug.SliceImage(z["slices"][i], float(z["spacing"]),
                            ug.ProbePose(z["rot"][i], z["trans"][i]))
              for i in range(len(z["slices"]))]
    return ug.SliceDataset(slices)


def _config(batch, densify):
    import paper_2505_05643_b200 as ug
    return ug.TrainConfig(n_gaussians=400, iterations=ITERS, seed=3, batch=batch,
                          heuristic_interval=densify, eval_interval=ITERS)


def _params(cloud):
    return {k: getattr(cloud, k).cpu().numpy() for k in
            ("means", "l_raw", "intensity_raw", "opacity_raw")} | {
        "bg": np.array([cloud.bg_intensity_raw, cloud.bg_opacity_raw])}


def _worker(rank, world, port, densify, q, peer=False, flags=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      UGS_PEER_UPDATE="1" if peer else "0",
                      UGS_PEER_FLAGS="1" if flags else "0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2505_05643_b200 as ug
        torch.cuda.set_device(0)
        cloud, _ = ug.train(_dataset(), _config(B, densify), device="cuda:0")
        q.put((rank, _params(cloud)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_two(densify, peer=False, flags=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, densify, q, peer, flags))
             for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, params = q.get(timeout=600)
        out[r] = params
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def test_two_ranks_match_single_process_global_batch():
    import paper_2505_05643_b200 as ug
    out = _run_two(densify=0)
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k      # replicas in lock-step
    ref, _ = ug.train(_dataset(), _config(2 * B, 0), device="cuda:0")
    ref = _params(ref)
    for k in ref:
        np.testing.assert_allclose(out[0][k], ref[k], rtol=1e-3, atol=1e-4, err_msg=k)


def test_two_ranks_densify_in_lockstep():
    out = _run_two(densify=5)
    assert out[0]["means"].shape == out[1]["means"].shape
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k


def test_peer_update_matches_single_process_global_batch():
    """The fused reduce-scatter + Adam + all-gather over CUDA IPC peer memory
    (ugs_peer_update): replicas identical, same trajectory as one process
    with the global batch."""
    import paper_2505_05643_b200 as ug
    out = _run_two(densify=0, peer=True)
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k
    ref, _ = ug.train(_dataset(), _config(2 * B, 0), device="cuda:0")
    ref = _params(ref)
    for k in ref:
        np.testing.assert_allclose(out[0][k], ref[k], rtol=1e-3, atol=1e-4, err_msg=k)


def test_peer_update_densify_in_lockstep():
    out = _run_two(densify=5, peer=True)
    ref = _run_two(densify=5, peer=False)
    assert out[0]["means"].shape == out[1]["means"].shape == ref[0]["means"].shape
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k
        np.testing.assert_allclose(out[0][k], ref[0][k], rtol=1e-3, atol=1e-4, err_msg=k)


def test_peer_device_barriers_match_collective_barriers():
    """The step barriers as device flags in the peer arenas (ugs_peer_signal
    / ugs_peer_update(epoch) / ugs_peer_wait) give bitwise the trajectory of
    the NCCL-style host barriers; n = 400 leaves the last rank a partial
    warp (the shard tail path of the coalesced all-gather)."""
    a = _run_two(densify=0, peer=True, flags=True)
    b = _run_two(densify=0, peer=True, flags=False)
    for k in a[0]:
        assert np.array_equal(a[0][k], b[0][k]), k
        assert np.array_equal(a[1][k], b[1][k]), k


def test_bench_two_ranks_one_device():
    """bench.py's N > 1 path end to end: two ranks on the one GPU over gloo
    (UGS_BENCH_ONE_DEVICE=1), fused peer update with device barriers; one
    JSON line from rank 0 with n_gpus = 2 (a functional check, not a
    measurement)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UGS_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--n-gaussians", "200000", "--no-tts", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2")
