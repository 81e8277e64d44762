"""CPU tests of bench.py's multi-GPU dispatch (no GPU work is started)."""
import sys

import pytest

from conftest import ROOT  # noqa: F401  (puts the repo on sys.path)


def test_self_launch_runs_one_rank_per_gpu_on_loopback(monkeypatch):
    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--workload", "tiny"])
    bench.self_launch(4)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--workload", "tiny"]


@pytest.mark.parametrize("env,expect", [({}, "group"), ({"VLQ_MULTI": "procs"}, "launch")])
def test_gpus_n_dispatch(monkeypatch, env, expect):
    """--gpus N without torchrun: the one-process group path by default (all N
    GPUs behind vlq_group), or one process per GPU under torch.distributed.run
    with VLQ_MULTI=procs; under torchrun WORLD_SIZE must equal N."""
    import bench
    for k in ("WORLD_SIZE", "RANK", "VLQ_MULTI"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    calls = []
    monkeypatch.setattr(bench, "run_group", lambda args, rank, world: calls.append(("group", args.gpus, rank, world)))
    monkeypatch.setattr(bench, "self_launch", lambda n: calls.append(("launch", n)) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--workload", "tiny"])
    if expect == "launch":
        with pytest.raises(SystemExit):
            bench.main()
        assert calls == [("launch", 2)]
    else:
        bench.main()
        assert calls == [("group", 2, 0, 1)]


def test_world_size_must_match_gpus(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--workload", "tiny"])
    with pytest.raises(SystemExit, match="WORLD_SIZE=4"):
        bench.main()
