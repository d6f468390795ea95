"""HuggingFace linear-layer replacement: RSRLinear and replace_linear_with_rsr.

The RSR-core paper's HF integration is not shipped by the
reference package, so this is designed new (SURVEY.md section
8b).  Numerics follow the reference's fused path (kernels.rsr_matvec_fused,
_native.py:339-353): per token, absmax-quantize the activation to int8
(float64 math, half away from zero), multiply exactly in the integer domain
against the ternarized weight, and dequantize by beta / scale -- one sm_100a
kernel per (stacked) linear.

Sibling linears that read the same input (q|k|v, gate|up) share ONE stacked
artifact (reference kernels.batched_preprocess, kernels.py:128-160); the
kernel applies each sibling's own beta per row, so every sibling's output is
bit-identical to running it alone.  The first sibling's call computes the
whole stack; the others consume its slices.
"""

from __future__ import annotations

import torch
from torch import nn

from .devicepack import ternarize_pack_device
from .kernels import batched_preprocess, fused_into, fused_rows_into

DEFAULT_K = 5  # fewest artifact bytes for BitNet-2B shapes


class RSRSiblingGroup:
    """One stacked artifact for linears that share an input."""

    def __init__(self, weights: list, k: int = DEFAULT_K, out_dtype=torch.bfloat16):
        dev = weights[0].device
        mats = [ternarize_pack_device(w) for w in weights]
        self.artifact, self.offsets = batched_preprocess(mats, k)
        self.betas = [m.weight_scale for m in mats]
        self.row_beta = torch.cat([
            torch.full((m.rows,), m.weight_scale, dtype=torch.float64, device=dev)
            for m in mats])
        self.in_features = mats[0].cols
        self.out_features = self.offsets[-1]
        self.out_dtype = out_dtype
        self.k = k
        self._out = None
        self._key = None
        self._pending: set = set()

    def compute(self, x2: torch.Tensor) -> torch.Tensor:
        """x2: (T, in) -> (T, sum(out)) in out_dtype.  One token (decode): one
        fused quantize/multiply/dequantize launch.  Several (prefill): the
        rows are quantized together, multiplied as one int8 batch and
        dequantized together -- each row bit-identical to the one-token path."""
        T = x2.shape[0]
        out = torch.empty(T, self.out_features, dtype=self.out_dtype, device=x2.device)
        if T == 1:
            fused_into(self.artifact, x2[0], out[0], beta=1.0, row_beta=self.row_beta)
        elif T > 1:
            fused_rows_into(self.artifact, x2, out, beta=1.0, row_beta=self.row_beta)
        return out

    def output_for(self, index: int, x2: torch.Tensor) -> torch.Tensor:
        """Sibling `index`'s slice of the stacked output for input x2.

        The first sibling to see a new input computes the whole stack; the
        others take their slices from it.  The stacked output is held only
        until every sibling has taken its slice (then dropped), and a new
        input -- or a sibling asking twice -- recomputes, so a stale result is
        never served."""
        key = (x2.data_ptr(), tuple(x2.shape), x2._version, x2.device)
        if self._out is not None and self._key == key and index in self._pending:
            out = self._out
            self._pending.discard(index)
        else:
            out = self.compute(x2)
            self._key = key
            self._pending = set(range(len(self.offsets) - 1)) - {index}
            self._out = out
        if not self._pending:
            self._out, self._key = None, None
        return out[:, self.offsets[index]:self.offsets[index + 1]]


class RSRLinear(nn.Module):
    """Drop-in for a bias-free nn.Linear whose weight is ternarized + RSR'd."""

    def __init__(self, group: RSRSiblingGroup, index: int):
        super().__init__()
        self.group = group
        self.index = index
        self.in_features = group.in_features
        self.out_features = group.offsets[index + 1] - group.offsets[index]

    @property
    def weight_scale(self) -> float:
        return self.group.betas[self.index]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        x2 = x.reshape(-1, shape[-1])
        if not x2.is_contiguous():
            x2 = x2.contiguous()
        y = self.group.output_for(self.index, x2)
        return y.reshape(*shape[:-1], self.out_features)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"k={self.group.k}, siblings={len(self.group.offsets) - 1}")


# sibling sets of the Llama/BitNet family (names under one parent module)
DEFAULT_SIBLINGS = (("q_proj", "k_proj", "v_proj"), ("gate_proj", "up_proj"))


def replace_linear_with_rsr(model: nn.Module, k: int = DEFAULT_K, sibling_groups=DEFAULT_SIBLINGS,
                            skip=("lm_head",), out_dtype=None) -> nn.Module:
    """Replace every bias-free nn.Linear (except `skip`) by an RSRLinear.

    Modeled on transformers' replace_with_bitnet_linear
    (transformers/integrations/bitnet.py:315-370).  Linears named in one
    tuple of `sibling_groups` under the same parent share a stacked artifact.
    The dense weights are released after conversion.
    """
    if out_dtype is None:
        out_dtype = next(model.parameters()).dtype
    converted = 0
    for parent in list(model.modules()):
        children = dict(parent.named_children())
        done = set()
        for names in sibling_groups:
            if all(isinstance(children.get(nm), nn.Linear) and children[nm].bias is None
                   and nm not in skip for nm in names):
                group = RSRSiblingGroup([children[nm].weight.data for nm in names], k, out_dtype)
                for i, nm in enumerate(names):
                    setattr(parent, nm, RSRLinear(group, i))
                    done.add(nm)
                    converted += 1
        for nm, ch in children.items():
            if nm in done or nm in skip or not isinstance(ch, nn.Linear) or ch.bias is not None:
                continue
            group = RSRSiblingGroup([ch.weight.data], k, out_dtype)
            setattr(parent, nm, RSRLinear(group, 0))
            converted += 1
    model._rsr_converted = converted
    torch.cuda.empty_cache()
    return model
