"""Sparse VGG / ResNet blocks built from the C-ABI layers.

PAPER.md L503 [§Evaluation] lists "VGG (a block of the VGG neural network)" and
"ResNet (a block of the ResNet neural network)" among the benchmarks; L507-509:
"We use the same sizes and parameters as in the original architectures ... block
10 in both ResNet and VGG"; Table 1 (L356-377) gives the per-layer densities.
Weights here are synthetic (random positions and values at those densities) —
the paper's LTH-pruned weights need training data we do not have.

Every layer runs in this library's kernels, with its elementwise tail fused into
the conv epilogue (operator fusion):

* ResNet basic block (inference, batch-norm folded into the bias):
  ``y = ReLU(conv2(ReLU(conv1(x) + b1)) + b2 + x)`` — two launches,
  ``spconv_forward_ex(RELU)`` then ``spconv_forward_ex(RELU | RESIDUAL)``.
* VGG block: ``conv + bias + ReLU`` for all but the last layer, then the fused
  ``conv + bias + ReLU + 2x2 max-pool`` (``spconv_fused_relu_maxpool``).

Python here only sequences launches and owns the intermediate buffers.
"""
from __future__ import annotations

from dataclasses import dataclass

from .spconv import SparseConv2d


@dataclass
class LayerSpec:
    C: int
    F: int
    density: float


# Table 1: ResNet-20 layers 9, 10 (a basic block of stage 2:
# 32 channels at 16x16 on CIFAR) and VGG-16 layers 8-10 (conv4_1..conv4_3: 256 ->
# 512 -> 512 channels at 28x28 on ImageNet, followed by the block's max-pool).
RESNET20_BLOCK10 = dict(H=16, W=16, layers=[LayerSpec(32, 32, 0.203), LayerSpec(32, 32, 0.161)])
VGG16_BLOCK10 = dict(H=28, W=28, layers=[LayerSpec(256, 512, 0.242), LayerSpec(512, 512, 0.058),
                                          LayerSpec(512, 512, 0.010)])


def make_layer(spec: LayerSpec, H: int, W: int, csr, bias, device=0, kernel="auto"):
    return SparseConv2d(spec.C, H, W, spec.F, 3, 1, 1, csr.rowptr, csr.colidx, csr.values, bias,
                        device=device, kernel=kernel)


class ResNetBasicBlock:
    """Two 3x3 same-size convs with folded batch norm and an identity shortcut."""

    def __init__(self, conv1: SparseConv2d, conv2: SparseConv2d):
        if conv1.F != conv2.C or conv2.F != conv1.C:
            raise ValueError("identity shortcut needs conv2.F == conv1.C")
        self.conv1, self.conv2 = conv1, conv2

    def forward(self, x, tmp=None, out=None, stream=None):
        y1 = self.conv1.forward_ex(x, relu=True, out=tmp, stream=stream)
        return self.conv2.forward_ex(y1, relu=True, residual=x, out=out, stream=stream)

    __call__ = forward

    def close(self):
        self.conv1.close()
        self.conv2.close()


class VGGBlock:
    """conv+ReLU, ..., conv+ReLU+maxpool (the pooled output and its argmax)."""

    def __init__(self, convs):
        if not convs:
            raise ValueError("empty block")
        for a, b in zip(convs, convs[1:]):
            if a.F != b.C:
                raise ValueError("channel mismatch between consecutive layers")
        self.convs = list(convs)

    def forward(self, x, stream=None, with_argmax=False):
        for conv in self.convs[:-1]:
            x = conv.forward_ex(x, relu=True, stream=stream)
        return self.convs[-1].fused_relu_maxpool(x, with_argmax=with_argmax, stream=stream)

    __call__ = forward

    def close(self):
        for c in self.convs:
            c.close()
