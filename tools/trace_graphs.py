"""Traces training-step dataflow graphs into the reference's graph format.

  python tools/trace_graphs.py            -> workloads/graphs/{resnet50_b32,bert_base_s512,gpt2_medium_s1024}.json.gz

One training step = forward + loss + backward + SGD update, traced with
``make_fx`` on FakeTensors (no memory, no data, random-init weights are never
materialised). Mapping onto memplan's model (graph.hpp:44-56):
  * every placeholder (input, label, parameter) is a node with role "source";
  * every aten op is a node ("weight_update" for the SGD update ops);
  * every op output tensor (and every placeholder value) is a data edge whose
    sinks are its consumer ops in program order; size = numel * itemsize;
    outputs nobody consumes (updated parameters, final values) are sinkless
    and stay resident to the end, exactly as in the reference;
  * getitem on multi-output ops is folded: each element is its own edge from
    the producing op; zero-byte values (empty shapes) are dropped.
Node order is the traced program order (topological).
"""
from __future__ import annotations

import gzip
import json
import os
import sys

import torch
from torch.fx.experimental.proxy_tensor import make_fx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "workloads", "graphs")


def _nbytes(v):
    if isinstance(v, torch.Tensor):
        return int(v.numel()) * v.element_size()
    return 0


def fx_to_memplan(gm: torch.fx.GraphModule, update_prefix="upd") -> dict:
    nodes, edges = [], []
    node_id = {}
    # value id -> (producer node id, size); lists for tuple outputs
    produced = {}
    users: dict[str, list[str]] = {}

    def add_edge(key, src, size):
        if size <= 0:
            return
        produced[key] = (src, size)
        users[key] = []

    count = 0
    for fx_node in gm.graph.nodes:
        if fx_node.op == "output":
            continue
        if fx_node.op == "get_attr":
            continue
        if fx_node.op == "call_function" and fx_node.target is __import__("operator").getitem:
            base, idx = fx_node.args
            key = f"{base.name}[{idx}]"
            if key in produced:
                produced[fx_node.name] = produced[key]
                users[fx_node.name] = users[key]
            continue
        nid = fx_node.name
        role = "compute"
        if fx_node.op == "placeholder":
            role = "source"
        elif str(fx_node.meta.get("memplan_role", "")) == "weight_update":
            role = "weight_update"
        nodes.append({"id": nid, "role": role})
        node_id[fx_node] = nid
        count += 1
        # consume inputs (each distinct value once per consumer)
        seen = set()
        for a in _flatten_args(fx_node):
            if a.name in users and a.name not in seen:
                seen.add(a.name)
                tgt = users[a.name]
                if nid not in tgt:
                    tgt.append(nid)
        val = fx_node.meta.get("val")
        if isinstance(val, (tuple, list)):
            for i, v in enumerate(val):
                add_edge(f"{nid}[{i}]", nid, _nbytes(v))
        else:
            add_edge(nid, nid, _nbytes(val))
    # edges in production order; aliases (getitem names) map to the same list
    emitted = set()
    for key, (src, size) in produced.items():
        if id(users[key]) in emitted:
            continue
        emitted.add(id(users[key]))
        edges.append({"id": "t_" + key.replace("[", "_").replace("]", ""), "source": src,
                      "sinks": users[key], "size": size, "kind": "data"})
    return {"nodes": nodes, "edges": edges}


def _flatten_args(fx_node):
    out = []

    def visit(x):
        if isinstance(x, torch.fx.Node):
            out.append(x)
        elif isinstance(x, (list, tuple)):
            for y in x:
                visit(y)
        elif isinstance(x, dict):
            for y in x.values():
                visit(y)
    visit(fx_node.args)
    visit(fx_node.kwargs)
    return out


def trace_train_step(model: torch.nn.Module, example_inputs: tuple, loss_fn) -> torch.fx.GraphModule:
    params = {k: v for k, v in model.named_parameters()}
    buffers = {k: v for k, v in model.named_buffers()}
    names = list(params)

    def step(param_list, buffer_list, *inputs):
        p = dict(zip(names, param_list))
        b = dict(zip(list(buffers), buffer_list))
        out = torch.func.functional_call(model, {**p, **b}, inputs[:-1])
        loss = loss_fn(out, inputs[-1])
        grads = torch.autograd.grad(loss, param_list)
        new = [w - 0.01 * g for w, g in zip(param_list, grads)]
        return loss, new

    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode(allow_non_fake_inputs=True) as mode:
        fp = [mode.from_tensor(v).requires_grad_(True) for v in params.values()]
        fb = [mode.from_tensor(v) for v in buffers.values()]
        fi = [mode.from_tensor(x) for x in example_inputs]
        gm = make_fx(step, tracing_mode="fake")(fp, fb, *fi)
    # mark the SGD update ops (sub of a parameter by a scaled gradient)
    outs = list(gm.graph.nodes)[-1].args[0]
    flat = []

    def visit(x):
        if isinstance(x, (list, tuple)):
            for y in x:
                visit(y)
        else:
            flat.append(x)
    visit(outs)
    for n in flat[1:]:  # flat[0] is the loss; the rest are the updated parameters
        if isinstance(n, torch.fx.Node):
            n.meta["memplan_role"] = "weight_update"
    return gm


def resnet50(batch=32):
    import torchvision
    m = torchvision.models.resnet50()
    m.eval()  # eval-mode BN keeps the graph free of running-stat updates
    x = torch.randn(batch, 3, 224, 224)
    y = torch.randint(0, 1000, (batch,))
    return m, (x, y), torch.nn.functional.cross_entropy


def bert_base(seq=512):
    from transformers import BertConfig, BertForMaskedLM
    cfg = BertConfig(attn_implementation="eager")
    m = BertForMaskedLM(cfg)
    m.eval()
    ids = torch.randint(0, cfg.vocab_size, (1, seq))

    def loss(out, y):
        logits = out.logits if hasattr(out, "logits") else out[0]
        return torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), y.view(-1))
    return m, (ids, ids.clone()), loss


class GPT2Block(torch.nn.Module):
    def __init__(self, d, h):
        super().__init__()
        self.ln1 = torch.nn.LayerNorm(d)
        self.qkv = torch.nn.Linear(d, 3 * d)
        self.proj = torch.nn.Linear(d, d)
        self.ln2 = torch.nn.LayerNorm(d)
        self.fc = torch.nn.Linear(d, 4 * d)
        self.out = torch.nn.Linear(4 * d, d)
        self.h = h

    def forward(self, x):
        b, s, d = x.shape
        q, k, v = self.qkv(self.ln1(x)).split(d, dim=-1)
        q = q.view(b, s, self.h, d // self.h).transpose(1, 2)
        k = k.view(b, s, self.h, d // self.h).transpose(1, 2)
        v = v.view(b, s, self.h, d // self.h).transpose(1, 2)
        att = (q @ k.transpose(-2, -1)) / (d // self.h) ** 0.5
        mask = torch.ones(s, s, dtype=torch.bool, device=x.device).tril()
        att = att.masked_fill(~mask, float("-inf")).softmax(-1)
        y = (att @ v).transpose(1, 2).reshape(b, s, d)
        x = x + self.proj(y)
        return x + self.out(torch.nn.functional.gelu(self.fc(self.ln2(x))))


class GPT2(torch.nn.Module):
    """GPT-2 medium (24 layers, d=1024, 16 heads) in plain torch."""

    def __init__(self, layers=24, d=1024, heads=16, vocab=50257, ctx=1024):
        super().__init__()
        self.wte = torch.nn.Embedding(vocab, d)
        self.wpe = torch.nn.Embedding(ctx, d)
        self.blocks = torch.nn.ModuleList([GPT2Block(d, heads) for _ in range(layers)])
        self.ln = torch.nn.LayerNorm(d)

    def forward(self, ids):
        pos = torch.arange(ids.shape[1], device=ids.device)
        x = self.wte(ids) + self.wpe(pos)
        for blk in self.blocks:
            x = blk(x)
        return self.ln(x) @ self.wte.weight.t()


def gpt2_medium(seq=1024):
    m = GPT2()
    ids = torch.randint(0, 50257, (1, seq))

    def loss(logits, y):
        return torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), y.view(-1))
    return m, (ids, ids.clone()), loss


MODELS = {"resnet50_b32": resnet50, "bert_base_s512": bert_base, "gpt2_medium_s1024": gpt2_medium}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        m, inputs, loss = MODELS[name]()
        gm = trace_train_step(m, inputs, loss)
        doc = fx_to_memplan(gm)
        path = os.path.join(OUT, name + ".json.gz")
        with gzip.open(path, "wt") as f:
            json.dump(doc, f, indent=2)
            f.write("\n")
        tb = sum(e["size"] for e in doc["edges"])
        print(f"{name}: {len(doc['nodes'])} nodes, {len(doc['edges'])} edges, "
              f"{sum(len(e['sinks']) for e in doc['edges'])} sinks, {tb / 2**30:.2f} GiB -> {path}")


if __name__ == "__main__":
    main(sys.argv[1:] or list(MODELS))
