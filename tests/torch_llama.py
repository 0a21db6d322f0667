"""A Llama-style decoder written as a plain PyTorch model (nn.Linear,
nn.RMSNorm, the torch.ops.opflow operators) — the user-side model the
TorchDynamo frontend (paper_2605_21603_b200/dynamo.py) compiles."""
import torch
import torch.nn as nn

from paper_2605_21603_b200 import dynamo as dyn


class Attention(nn.Module):
    def __init__(self, hidden, heads, kv_heads, head_dim, seq_len, theta=500000.0):
        super().__init__()
        self.heads, self.kv_heads, self.head_dim, self.seq_len, self.theta = heads, kv_heads, head_dim, seq_len, theta
        self.qkv = nn.Linear(hidden, (heads + 2 * kv_heads) * head_dim, bias=False)
        self.o = nn.Linear(heads * head_dim, hidden, bias=False)

    def forward(self, h, positions):
        qkv = self.qkv(h)
        qkv = torch.ops.opflow.rope(qkv, positions, self.heads, self.kv_heads, self.head_dim, self.theta)
        ctx = torch.ops.opflow.attn_prefill(qkv, self.heads, self.kv_heads, self.head_dim, self.seq_len)
        return self.o(ctx)


class MLP(nn.Module):
    def __init__(self, hidden, inter):
        super().__init__()
        self.gate_up = nn.Linear(hidden, 2 * inter, bias=False)
        self.down = nn.Linear(inter, hidden, bias=False)

    def forward(self, h):
        return self.down(torch.ops.opflow.silu_mul(self.gate_up(h)))


class Block(nn.Module):
    def __init__(self, hidden, heads, kv_heads, head_dim, inter, seq_len, eps=1e-5, idx=0):
        super().__init__()
        self.idx = idx
        self.attn_norm = nn.RMSNorm(hidden, eps=eps)
        self.attn = Attention(hidden, heads, kv_heads, head_dim, seq_len)
        self.mlp_norm = nn.RMSNorm(hidden, eps=eps)
        self.mlp = MLP(hidden, inter)

    def forward(self, x, positions):
        x = x + self.attn(self.attn_norm(x), positions)
        with dyn.mark(f"ffn{self.idx}"):
            h = self.mlp_norm(x)
        return x + self.mlp(h)


class Llama(nn.Module):
    def __init__(self, layers=2, hidden=512, heads=4, kv_heads=2, head_dim=128, inter=1024, seq_len=128):
        super().__init__()
        self.layers = nn.ModuleList([Block(hidden, heads, kv_heads, head_dim, inter, seq_len, idx=i) for i in range(layers)])

    def forward(self, x, positions):
        for layer in self.layers:
            x = layer(x, positions)
        return x


def init_(model, seed=0):
    g = torch.Generator().manual_seed(seed)
    with torch.no_grad():
        for name, p in model.named_parameters():
            if name.endswith("norm.weight"):
                p.copy_(1.0 + 0.1 * (torch.rand(p.shape, generator=g) - 0.5))
            else:
                p.copy_((torch.rand(p.shape, generator=g) * 2 - 1) / p.shape[1] ** 0.5)
    return model
