"""Operator-graph and topology generators used as synthetic inputs.

The first group reproduces the reference's example families graph-for-graph
(same op ids, shapes, edges and parameter bytes -- reference
``pkg/src/parasim/models.py:167-271``) so that results are comparable on
identical inputs.  The second group builds the benchmark shapes the
reference does not ship: Inception-v3 (125 ops with a
1x1 input source), ResNet-101 (141 ops) and a seeded random DAG that covers
all eight operator kinds.  Everything here is host-side input data.
"""

from __future__ import annotations

import random

from .graph import DeviceTopology, Operation, OperatorGraph, OperatorKind, conv_out_size, \
    parallelizable_dims, shape
from .partition import ParallelizationConfig, ParallelizationStrategy

__all__ = [
    "rnn3", "lenet_like", "alexnet_like", "rnnlm_like", "rnntc_like", "nmt_like",
    "single_node_topology", "multi_node_topology", "rnn3_model_parallel_strategy",
    "MODEL_GENERATORS", "TOPOLOGY_GENERATORS",
    "inception_v3", "resnet101", "random_dag",
]

F32 = 4


# -- builders ----------------------------------------------------------------

class _Builder:
    """Small helper that appends ops/edges in a fixed order."""

    def __init__(self, g: OperatorGraph | None = None):
        self.g = g if g is not None else OperatorGraph()

    def out(self, op_id):
        return self.g.ops[op_id].output_shape

    def embedding(self, op_id, batch, hidden, vocab):
        self.g.add_op(Operation(op_id, OperatorKind("Embedding", {"vocab_size": vocab}),
                                (shape(("sample", batch)),),
                                shape(("sample", batch), ("channel", hidden)),
                                param_bytes=vocab * hidden * F32))
        return op_id

    def matmul(self, op_id, src, cout, with_params=True):
        s = self.out(src)
        feats = s.volume() // s.size("sample")
        self.g.add_op(Operation(op_id, OperatorKind("MatMul"), (s,),
                                shape(("sample", s.size("sample")), ("channel", cout)),
                                param_bytes=feats * cout * F32 if with_params else 0))
        self.g.add_tensor(src, op_id)
        return op_id

    def elementwise(self, op_id, srcs):
        s = self.out(srcs[0])
        self.g.add_op(Operation(op_id, OperatorKind("ElementWise"), (s,) * len(srcs), s))
        for slot, src in enumerate(srcs):
            self.g.add_tensor(src, op_id, dst_slot=slot)
        return op_id

    def _window(self, tag, op_id, src, kh, kw, sh, sw, padding, cout=None, in_shape=None):
        s = in_shape if in_shape is not None else self.out(src)
        oh = conv_out_size(s.size("height"), kh, sh, padding)
        ow = conv_out_size(s.size("width"), kw, sw, padding)
        cin = s.size("channel")
        cout = cin if cout is None else cout
        hp = {"kernel_h": kh, "kernel_w": kw, "stride_h": sh, "stride_w": sw, "padding": padding}
        params = cin * kh * kw * cout * F32 if tag == "Conv2D" else 0
        self.g.add_op(Operation(op_id, OperatorKind(tag, hp), (s,),
                                shape(("sample", s.size("sample")), ("height", oh),
                                      ("width", ow), ("channel", cout)),
                                param_bytes=params))
        if in_shape is None:
            self.g.add_tensor(src, op_id)
        return op_id

    def conv2d(self, op_id, src, cout, kh=3, kw=None, stride=1, padding="same", in_shape=None):
        kw = kh if kw is None else kw
        return self._window("Conv2D", op_id, src, kh, kw, stride, stride, padding, cout, in_shape)

    def pool2d(self, op_id, src, k=2, stride=2, padding="valid"):
        return self._window("Pool2D", op_id, src, k, k, stride, stride, padding)

    def concat(self, op_id, srcs, axis="channel"):
        shapes = [self.out(s) for s in srcs]
        base = shapes[0]
        total = sum(s.size(axis) for s in shapes)
        out = shape(*((n, total if n == axis else sz) for n, sz in base.dims),
                    element_size=base.element_size)
        self.g.add_op(Operation(op_id, OperatorKind("Concat", {"axis": axis}), tuple(shapes), out))
        for slot, src in enumerate(srcs):
            self.g.add_tensor(src, op_id, dst_slot=slot)
        return op_id

    def recurrent(self, prefix, steps, layers, feed, hidden):
        tops = []
        for t in range(steps):
            below = feed(t)
            for layer in range(layers):
                mm, cell = f"{prefix}_mm{layer}_{t}", f"{prefix}_cell{layer}_{t}"
                self.matmul(mm, below, hidden)
                self.elementwise(cell, [mm] if t == 0 else [mm, f"{prefix}_cell{layer}_{t - 1}"])
                below = cell
            tops.append(below)
        return tops


# -- the reference's families (identical graphs) -------------------------------

def rnn3(steps=2, batch=32, hidden=32, vocab=64) -> OperatorGraph:
    b = _Builder()
    for t in range(steps):
        b.embedding(f"embed{t}", batch, hidden, vocab)
    for t, top in enumerate(b.recurrent("rec", steps, 1, lambda t: f"embed{t}", hidden)):
        b.matmul(f"out{t}", top, vocab)
    return b.g


def rnn3_model_parallel_strategy(g: OperatorGraph, topo: DeviceTopology) -> ParallelizationStrategy:
    """embed* / rec* / everything else pinned unsplit to devices 0 / 1 / 2."""
    devs = topo.device_ids()
    if len(devs) < 3:
        raise ValueError("rnn3 model parallelism needs at least 3 devices")
    configs = {}
    for op_id, op in g.ops.items():
        layer = 0 if op_id.startswith("embed") else 1 if op_id.startswith("rec") else 2
        configs[op_id] = ParallelizationConfig(dict.fromkeys(parallelizable_dims(op), 1),
                                               (devs[layer],))
    return ParallelizationStrategy(configs)


def _first_conv(b, op_id, batch, image, cin, cout):
    b.conv2d(op_id, None, cout, 3, padding="same",
             in_shape=shape(("sample", batch), ("height", image), ("width", image),
                            ("channel", cin)))


def lenet_like(batch=4, image=8, in_channels=2, conv_channels=(4, 8), fc_hidden=16,
               classes=8) -> OperatorGraph:
    b = _Builder()
    _first_conv(b, "conv1", batch, image, in_channels, conv_channels[0])
    b.pool2d("pool1", "conv1")
    b.conv2d("conv2", "pool1", conv_channels[1])
    b.pool2d("pool2", "conv2")
    b.matmul("fc1", "pool2", fc_hidden)
    b.matmul("fc2", "fc1", classes)
    return b.g


def alexnet_like(batch=16, image=16, in_channels=3, base_channels=8, fc_hidden=64,
                 classes=16) -> OperatorGraph:
    c = base_channels
    b = _Builder()
    _first_conv(b, "conv1", batch, image, in_channels, c)
    b.pool2d("pool1", "conv1")
    b.conv2d("conv2", "pool1", 2 * c)
    b.pool2d("pool2", "conv2")
    b.conv2d("conv3", "pool2", 4 * c)
    b.conv2d("conv4", "conv3", 4 * c)
    b.conv2d("conv5", "conv4", 2 * c)
    b.pool2d("pool3", "conv5")
    b.matmul("fc1", "pool3", fc_hidden)
    b.matmul("fc2", "fc1", fc_hidden)
    b.matmul("fc3", "fc2", classes)
    return b.g


def rnnlm_like(steps=2, layers=2, batch=16, hidden=32, vocab=64) -> OperatorGraph:
    b = _Builder()
    for t in range(steps):
        b.embedding(f"embed{t}", batch, hidden, vocab)
    for t, top in enumerate(b.recurrent("lm", steps, layers, lambda t: f"embed{t}", hidden)):
        b.matmul(f"softmax{t}", top, vocab)
    return b.g


def rnntc_like(steps=4, layers=4, batch=16, hidden=32, vocab=64, classes=8) -> OperatorGraph:
    b = _Builder()
    for t in range(steps):
        b.embedding(f"embed{t}", batch, hidden, vocab)
    tops = b.recurrent("tc", steps, layers, lambda t: f"embed{t}", hidden)
    b.matmul("classifier", tops[-1], classes)
    return b.g


def nmt_like(steps=4, layers=2, batch=16, hidden=32, vocab=64) -> OperatorGraph:
    b = _Builder()
    for t in range(steps):
        b.embedding(f"enc_embed{t}", batch, hidden, vocab)
    context = b.recurrent("enc", steps, layers, lambda t: f"enc_embed{t}", hidden)[-1]
    for t in range(steps):
        b.embedding(f"dec_embed{t}", batch, hidden, vocab)
    for t, top in enumerate(b.recurrent("dec", steps, layers, lambda t: f"dec_embed{t}", hidden)):
        b.matmul(f"att_mm{t}", top, hidden)
        b.elementwise(f"att{t}", [f"att_mm{t}", context])
        b.matmul(f"softmax{t}", f"att{t}", vocab)
    return b.g


def single_node_topology(gpus=4, bandwidth=32e9, latency=1e-6, kind="gpu") -> DeviceTopology:
    topo = DeviceTopology()
    ids = [f"gpu{i:02d}" for i in range(gpus)]
    for dev in ids:
        topo.add_device(dev, kind, "node00")
    for i in range(len(ids)):
        for j in range(i + 1, len(ids)):
            topo.add_connection(ids[i], ids[j], bandwidth, latency)
    return topo


def multi_node_topology(nodes=2, gpus_per_node=4, intra_bandwidth=16e9, inter_bandwidth=7e9,
                        intra_latency=1e-6, inter_latency=5e-6, kind="gpu") -> DeviceTopology:
    topo = DeviceTopology()
    placed = []
    for n in range(nodes):
        for i in range(gpus_per_node):
            dev = f"n{n:02d}g{i}"
            topo.add_device(dev, kind, f"node{n:02d}")
            placed.append((n, dev))
    for x in range(len(placed)):
        for y in range(x + 1, len(placed)):
            (na, a), (nb, b) = placed[x], placed[y]
            same = na == nb
            topo.add_connection(a, b, intra_bandwidth if same else inter_bandwidth,
                                intra_latency if same else inter_latency)
    return topo


MODEL_GENERATORS = {
    "rnn3": rnn3, "lenet-like": lenet_like, "alexnet-like": alexnet_like,
    "rnnlm-like": rnnlm_like, "rnntc-like": rnntc_like, "nmt-like": nmt_like,
}
TOPOLOGY_GENERATORS = {"p100-node": single_node_topology, "k80-cluster": multi_node_topology}


# -- benchmark shapes the reference lacks ----------------------

def _input_source(b, batch, side, channels):
    """1x1/1 parameterless Pool2D standing in for the image input."""
    b._window("Pool2D", "input", None, 1, 1, 1, 1, "valid",
              in_shape=shape(("sample", batch), ("height", side), ("width", side),
                             ("channel", channels)))
    return "input"


def inception_v3(batch=64, image=299, classes=1000) -> OperatorGraph:
    """torchvision Inception-v3 topology (BN/ReLU folded, aux head omitted):
    stem, 3xA, B, 4xC, D, 2xE, global pool, fc -- 125 ops."""
    b = _Builder()
    x = _input_source(b, batch, image, 3)
    x = b.conv2d("stem_c1", x, 32, 3, stride=2, padding="valid")
    x = b.conv2d("stem_c2", x, 32, 3, padding="valid")
    x = b.conv2d("stem_c3", x, 64, 3, padding="same")
    x = b.pool2d("stem_p1", x, 3, 2, "valid")
    x = b.conv2d("stem_c4", x, 80, 1)
    x = b.conv2d("stem_c5", x, 192, 3, padding="valid")
    x = b.pool2d("stem_p2", x, 3, 2, "valid")

    def block_a(p, x, pool_features):
        b1 = b.conv2d(f"{p}_b1", x, 64, 1)
        b5 = b.conv2d(f"{p}_b5a", x, 48, 1)
        b5 = b.conv2d(f"{p}_b5b", b5, 64, 5)
        b3 = b.conv2d(f"{p}_b3a", x, 64, 1)
        b3 = b.conv2d(f"{p}_b3b", b3, 96, 3)
        b3 = b.conv2d(f"{p}_b3c", b3, 96, 3)
        bp = b.pool2d(f"{p}_bpp", x, 3, 1, "same")
        bp = b.conv2d(f"{p}_bpc", bp, pool_features, 1)
        return b.concat(f"{p}_cat", [b1, b5, b3, bp])

    def block_b(p, x):
        b3 = b.conv2d(f"{p}_b3", x, 384, 3, stride=2, padding="valid")
        bd = b.conv2d(f"{p}_bda", x, 64, 1)
        bd = b.conv2d(f"{p}_bdb", bd, 96, 3)
        bd = b.conv2d(f"{p}_bdc", bd, 96, 3, stride=2, padding="valid")
        bp = b.pool2d(f"{p}_bp", x, 3, 2, "valid")
        return b.concat(f"{p}_cat", [b3, bd, bp])

    def block_c(p, x, c7):
        b1 = b.conv2d(f"{p}_b1", x, 192, 1)
        s = b.conv2d(f"{p}_b7a", x, c7, 1)
        s = b.conv2d(f"{p}_b7b", s, c7, 1, 7)
        s = b.conv2d(f"{p}_b7c", s, 192, 7, 1)
        d = b.conv2d(f"{p}_bda", x, c7, 1)
        d = b.conv2d(f"{p}_bdb", d, c7, 7, 1)
        d = b.conv2d(f"{p}_bdc", d, c7, 1, 7)
        d = b.conv2d(f"{p}_bdd", d, c7, 7, 1)
        d = b.conv2d(f"{p}_bde", d, 192, 1, 7)
        bp = b.pool2d(f"{p}_bpp", x, 3, 1, "same")
        bp = b.conv2d(f"{p}_bpc", bp, 192, 1)
        return b.concat(f"{p}_cat", [b1, s, d, bp])

    def block_d(p, x):
        b3 = b.conv2d(f"{p}_b3a", x, 192, 1)
        b3 = b.conv2d(f"{p}_b3b", b3, 320, 3, stride=2, padding="valid")
        b7 = b.conv2d(f"{p}_b7a", x, 192, 1)
        b7 = b.conv2d(f"{p}_b7b", b7, 192, 1, 7)
        b7 = b.conv2d(f"{p}_b7c", b7, 192, 7, 1)
        b7 = b.conv2d(f"{p}_b7d", b7, 192, 3, stride=2, padding="valid")
        bp = b.pool2d(f"{p}_bp", x, 3, 2, "valid")
        return b.concat(f"{p}_cat", [b3, b7, bp])

    def block_e(p, x):
        b1 = b.conv2d(f"{p}_b1", x, 320, 1)
        t = b.conv2d(f"{p}_b3a", x, 384, 1)
        t = b.concat(f"{p}_b3cat", [b.conv2d(f"{p}_b3b", t, 384, 1, 3),
                                    b.conv2d(f"{p}_b3c", t, 384, 3, 1)])
        d = b.conv2d(f"{p}_bda", x, 448, 1)
        d = b.conv2d(f"{p}_bdb", d, 384, 3)
        d = b.concat(f"{p}_bdcat", [b.conv2d(f"{p}_bdc", d, 384, 1, 3),
                                    b.conv2d(f"{p}_bdd", d, 384, 3, 1)])
        bp = b.pool2d(f"{p}_bpp", x, 3, 1, "same")
        bp = b.conv2d(f"{p}_bpc", bp, 192, 1)
        return b.concat(f"{p}_cat", [b1, t, d, bp])

    for i, pf in enumerate((32, 64, 64)):
        x = block_a(f"a{i}", x, pf)
    x = block_b("b0", x)
    for i, c7 in enumerate((128, 160, 160, 192)):
        x = block_c(f"c{i}", x, c7)
    x = block_d("d0", x)
    for i in range(2):
        x = block_e(f"e{i}", x)
    x = b.pool2d("head_pool", x, 8, 8, "valid")
    b.matmul("head_fc", x, classes)
    return b.g


def resnet101(batch=64, image=224, classes=1000, stages=(3, 4, 23, 3)) -> OperatorGraph:
    """Bottleneck ResNet-101: stem, four stages, global pool, fc -- 141 ops."""
    b = _Builder()
    x = _input_source(b, batch, image, 3)
    x = b.conv2d("stem_conv", x, 64, 7, stride=2, padding="same")
    x = b.pool2d("stem_pool", x, 3, 2, "same")
    for si, (blocks, width) in enumerate(zip(stages, (64, 128, 256, 512))):
        for bi in range(blocks):
            p = f"s{si}b{bi:02d}"
            stride = 2 if (bi == 0 and si > 0) else 1
            y = b.conv2d(f"{p}_c1", x, width, 1)
            y = b.conv2d(f"{p}_c2", y, width, 3, stride=stride, padding="same")
            y = b.conv2d(f"{p}_c3", y, 4 * width, 1)
            skip = b.conv2d(f"{p}_proj", x, 4 * width, 1, stride=stride) if bi == 0 else x
            x = b.elementwise(f"{p}_add", [y, skip])
    x = b.pool2d("head_pool", x, 7, 7, "valid")
    b.matmul("head_fc", x, classes)
    return b.g


def random_dag(n_ops: int, seed: int = 0, batch_choices=(2, 4, 8)) -> OperatorGraph:
    """Seeded random DAG over all eight kinds, grown by attaching each new op
    to a uniformly chosen earlier op (plus a same-shape partner for the
    2-input kinds).  O(n) expected: partners are found through shape buckets."""
    rng = random.Random(seed)
    b = _Builder()
    by_shape: dict = {}
    by_sig: dict = {}
    avail: list[str] = []

    def register(op_id):
        avail.append(op_id)
        s = b.out(op_id)
        by_shape.setdefault(s, []).append(op_id)
        if s.has("channel"):
            sig = tuple((n, sz) for n, sz in s.dims if n != "channel")
            by_sig.setdefault(sig, []).append(op_id)

    def source(op_id):
        batch = rng.choice(batch_choices)
        flavor = rng.choice(("embed", "vector", "image", "sequence"))
        g = b.g
        if flavor == "embed":
            b.embedding(op_id, batch, rng.choice((4, 8)), rng.choice((8, 16)))
        elif flavor == "vector":
            cin, cout = rng.choice((4, 8)), rng.choice((4, 8, 16))
            g.add_op(Operation(op_id, OperatorKind("MatMul"), (shape(("sample", batch), ("channel", cin)),),
                               shape(("sample", batch), ("channel", cout)), param_bytes=cin * cout * F32))
        elif flavor == "image":
            side = rng.choice((4, 8))
            b.conv2d(op_id, None, rng.choice((2, 4)), 3,
                     in_shape=shape(("sample", batch), ("height", side), ("width", side),
                                    ("channel", rng.choice((1, 2)))))
        else:
            length, cin, cout = rng.choice((4, 8, 16)), rng.choice((2, 4)), rng.choice((2, 4))
            g.add_op(Operation(op_id, OperatorKind("Conv1D", {"kernel": 3, "stride": 1, "padding": "same"}),
                               (shape(("sample", batch), ("length", length), ("channel", cin)),),
                               shape(("sample", batch), ("length", length), ("channel", cout)),
                               param_bytes=cin * 3 * cout * F32))
        register(op_id)

    def grow(op_id):
        src = rng.choice(avail)
        s = b.out(src)
        names = s.names()
        moves = ["matmul", "elementwise"]
        if "height" in names:
            moves.append("conv2d")
            if s.size("height") % 2 == 0 and s.size("width") % 2 == 0:
                moves.append("pool2d")
        elif "length" in names:
            moves.append("conv1d")
            if s.size("length") % 2 == 0:
                moves.append("pool1d")
        twins = [o for o in by_shape.get(s, ()) if o != src]
        if twins:
            moves.append("elementwise2")
        mates = []
        if "channel" in names:
            sig = tuple((n, sz) for n, sz in s.dims if n != "channel")
            mates = [o for o in by_sig.get(sig, ()) if o != src]
        if mates:
            moves.append("concat")
        move = rng.choice(moves)
        g = b.g
        if move == "matmul":
            b.matmul(op_id, src, rng.choice((4, 8, 16)))
        elif move == "elementwise":
            b.elementwise(op_id, [src])
        elif move == "elementwise2":
            b.elementwise(op_id, [src, rng.choice(twins)])
        elif move == "concat":
            b.concat(op_id, [src, rng.choice(mates)])
        elif move == "conv2d":
            b.conv2d(op_id, src, rng.choice((2, 4, 8)), 3)
        elif move == "pool2d":
            b.pool2d(op_id, src, 2, 2, "valid")
        elif move == "conv1d":
            cout = rng.choice((2, 4, 8))
            g.add_op(Operation(op_id, OperatorKind("Conv1D", {"kernel": 3, "stride": 1, "padding": "same"}),
                               (s,), shape(("sample", s.size("sample")), ("length", s.size("length")),
                                           ("channel", cout)),
                               param_bytes=s.size("channel") * 3 * cout * F32))
            g.add_tensor(src, op_id)
        else:
            g.add_op(Operation(op_id, OperatorKind("Pool1D", {"kernel": 2, "stride": 2, "padding": "valid"}),
                               (s,), shape(("sample", s.size("sample")),
                                           ("length", conv_out_size(s.size("length"), 2, 2, "valid")),
                                           ("channel", s.size("channel")))))
            g.add_tensor(src, op_id)
        register(op_id)

    width = len(str(max(n_ops, 10)))
    for i in range(rng.randint(1, 2)):
        source(f"src{i:0{width}d}")
    i = 0
    while len(b.g.ops) < n_ops:
        grow(f"op{i:0{width}d}")
        i += 1
    return b.g
