"""bench.py plumbing on CPU: the --gpus N self-launch and the JSON config block."""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def test_gpus_n_outside_torchrun_relaunches_under_torch_distributed_run(monkeypatch):
    import bench

    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--warmup", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_config_block_names_the_ranks_that_ran():
    import argparse

    import bench

    args = argparse.Namespace(config="llama8k_causal")
    blk1 = bench.config_block(bench.CONFIGS["llama8k_causal"], args, 1)
    blk8 = bench.config_block(bench.CONFIGS["llama8k_causal"], args, 8)
    assert blk1["parallelism"] == "single GPU"
    assert "8 GPUs" in blk8["parallelism"]
    assert "ma_source" not in blk1 and "kernel_ms" not in blk1
    for k in ("workload", "B", "Hq", "Hkv", "N", "D", "causal"):
        assert k in blk1
