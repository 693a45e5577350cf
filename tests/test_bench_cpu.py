"""bench.py contract pieces that need no GPU: the N>1 self-spawn command, the
reference arm's rank-0-only behaviour, and the CPU baseline's two-point fit."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_spawn_without_world_size(monkeypatch):
    """`python bench.py --gpus 4` with WORLD_SIZE unset launches 4 ranks
    through torch.distributed.run on 127.0.0.1 with the same arguments."""
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]


def test_reference_arm_other_ranks_exit_quietly(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "4"])
    bench.main()
    assert capsys.readouterr().out == ""


def test_cpu_fit_recovers_a_synthetic_cost():
    """T(M) = c + k F(M): two exact points give back c, k and the extrapolation."""
    smp = bench.CpuSample.__new__(bench.CpuSample)
    from oracle.model import llama_tiny_config
    smp.cfg = llama_tiny_config(n_layers=1, n_heads=32, n_kv_heads=8, head_dim=128,
                                ffn_dim=14336, vocab_size=256, max_seq=1024)
    smp.layers_model, smp.seq, smp.p = 32, 8192, 8
    c, k = 2.0, 1 / 50e9
    smp.times = {m: [c + k * smp.layer_flops(m)] for m in smp.POINTS}
    c2, k2, _, _, t_full = smp.fit()
    assert abs(c2 - c) < 1e-9 and abs(k2 - k) / k < 1e-9
    assert abs(t_full - 32 * (c + k * smp.layer_flops(8192))) < 1e-6
    d = smp.describe()
    assert d["kind"] == "port" and d["cores"] == 8 and "T(M) = c + k*F(M)" in d["sample"]
