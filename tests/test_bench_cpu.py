"""bench.py host logic (CPU): the `--gpus N` self-launch under
torch.distributed.run, the sharded scene split the ranks build, and the
per-kernel roofline table."""
import sys

import pytest

import bench


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse()
    assert args.config == "C4"                        # the sharded default at N > 1
    bench.relaunch_distributed(args)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_shards_cover_the_scene_once(world):
    got = []
    for r in range(world):
        local, keys, scaling, full = bench.scene_config("C4", r, world)
        assert scaling == "strong" and len(full.patches) == 8
        assert [k for _, k in keys] == list(range(sum(len(x) for x in got), sum(len(x) for x in got) + len(keys)))
        got.append(keys)
        assert local.fft_cascades == full.fft_cascades
    assert [k for ks in got for _, k in ks] == list(range(8))


def test_c3_weak_scaling_is_one_coherent_scene():
    a = bench.scene_config("C3", 0, 2)
    b = bench.scene_config("C3", 1, 2)
    assert a[0].seed == b[0].seed                     # same background on every rank
    assert a[1] == [(a[0].seed, 0)] and b[1] == [(a[0].seed, 1)]
    assert a[0].patches[0].origin != b[0].patches[0].origin


def test_roofline_names_the_longest_stage():
    stage = {"fft": 0.030, "advect": 0.022, "compose": 0.034, "smooth": 0.019, "frame": 0.1}
    units = {"fft": 1024.0 ** 2, "advect": 858e3, "compose": 1024.0 ** 2, "smooth": 2.6e6}
    r = bench.roofline(stage, units, 6551.4, {"config": "C3", "stages": {"compose": 123.0}}, "C3")
    assert r["kernel"] == "compose" and r["traffic"] == 123.0
    assert abs(r["achieved"] - 20.0 * 1024 ** 2 / 34e-6 / 1e9) < 1e-6
    assert set(r["per_kernel"]) == {"fft", "advect", "compose", "smooth"}
    assert bench.roofline(stage, units, 6551.4, {"config": "C3", "stages": {}}, "C4")["traffic"] is None
