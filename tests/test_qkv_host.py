"""Host-side layout of the fused projection GEMM's weight (ops.qkv_weight_permute): D/128 tiles of
128 q rows, then D/64 tiles of [64 k rows; the same channels' 64 v rows] (CPU, no kernel)."""

import pytest
import torch

from paper_2503_01868_b200 import ops


def test_qkv_weight_permute_layout():
    D = 256
    w = torch.arange(3 * D, dtype=torch.float32)[:, None].expand(3 * D, D).contiguous()  # row r holds r
    wp = ops.qkv_weight_permute(w)
    rows = wp[:, 0].long().tolist()
    assert rows[:D] == list(range(D))  # q rows in order
    for j in range(D // 64):
        blk = rows[D + 128 * j: D + 128 * (j + 1)]
        assert blk[:64] == [D + 64 * j + i for i in range(64)]      # k rows of channels 64j..
        assert blk[64:] == [2 * D + 64 * j + i for i in range(64)]  # v rows of the same channels
    assert sorted(rows) == list(range(3 * D))


def test_qkv_weight_permute_rejects():
    with pytest.raises(ValueError):
        ops.qkv_weight_permute(torch.zeros((3 * 96, 96)))
    with pytest.raises(ValueError):
        ops.qkv_weight_permute(torch.zeros((2 * 128, 128)))
