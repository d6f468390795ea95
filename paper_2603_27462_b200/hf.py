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
from .kernels import batched_preprocess, fused_into, fused_norm_into, fused_rows_into

DEFAULT_K = 5  # fewest artifact bytes for BitNet-2B shapes


def rms_norm_reference(x: torch.Tensor, weight: torch.Tensor, eps: float) -> torch.Tensor:
    """HF BitNetRMSNorm / LlamaRMSNorm arithmetic (fp32 mean of squares,
    x * rsqrt(mean + eps) rounded to the input dtype, times the weight)."""
    h = x.to(torch.float32)
    h = h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + eps)
    return weight * h.to(x.dtype)


class RSRSiblingGroup:
    """One stacked artifact for linears that share an input.

    With `norm` (an RMSNorm module whose output feeds only these linears)
    the group is a BitLinear: the norm runs inside the fused kernel's
    prologue (rsr_fused_matvec_norm) and the caller replaces the norm module
    by an identity.  Shapes the fused prologue cannot take fall back to the
    norm in torch followed by the plain fused kernel."""

    def __init__(self, weights: list, k: int = DEFAULT_K, out_dtype=torch.bfloat16, norm=None):
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
        self.norm_w = None if norm is None else \
            norm.weight.data.to(device=dev, dtype=torch.bfloat16).contiguous()
        self.norm_eps = 0.0 if norm is None else float(norm.variance_epsilon)
        # the fused kernel's register-staged prologue: one tile, n % 8 == 0,
        # at most 16 elements per thread of a 20-warp CTA
        self.norm_in_kernel = (self.in_features % 8 == 0 and self.in_features <= 10240
                               and self.artifact.plan.tile_count == 1)
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
        if self.norm_w is not None and x2.dtype != torch.bfloat16:
            x2 = rms_norm_reference(x2, self.norm_w.to(x2.dtype), self.norm_eps)
            norm = None
        else:
            norm = self.norm_w
        if T == 1:
            if norm is not None and self.norm_in_kernel:
                fused_norm_into(self.artifact, x2[0], out[0], norm, self.norm_eps, beta=1.0,
                                row_beta=self.row_beta)
                return out
            if norm is not None:
                x2 = rms_norm_reference(x2, norm, self.norm_eps)
            fused_into(self.artifact, x2[0], out[0], beta=1.0, row_beta=self.row_beta)
        elif T > 1:
            fused_rows_into(self.artifact, x2, out, beta=1.0, row_beta=self.row_beta,
                            norm_w=norm, norm_eps=self.norm_eps)
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

# BitNet decoder layer: RMSNorms whose output feeds only the listed linears
# (modeling_bitnet.py: BitNetDecoderLayer, BitNetAttention, BitNetMLP):
# (norm owner path, norm name, linears' parent path, linear names)
BITNET_NORMS = (("", "input_layernorm", "self_attn", ("q_proj", "k_proj", "v_proj")),
                ("", "post_attention_layernorm", "mlp", ("gate_proj", "up_proj")),
                ("self_attn", "attn_sub_norm", "self_attn", ("o_proj",)),
                ("mlp", "ffn_sub_norm", "mlp", ("down_proj",)))


def _sub(mod, path):
    for part in [p for p in path.split(".") if p]:
        mod = getattr(mod, part, None)
        if mod is None:
            return None
    return mod


def _norm_plan(model: nn.Module) -> dict:
    """{id(linear parent): {linear names tuple: (norm owner, norm name, norm)}}
    for every decoder layer that has the BitNet structure."""
    plan = {}
    for layer in model.modules():
        if not (hasattr(layer, "input_layernorm") and hasattr(layer, "self_attn")
                and hasattr(layer, "mlp")):
            continue
        for owner_path, norm_name, parent_path, names in BITNET_NORMS:
            owner, parent = _sub(layer, owner_path), _sub(layer, parent_path)
            norm = getattr(owner, norm_name, None) if owner is not None else None
            if norm is None or parent is None or not hasattr(norm, "variance_epsilon"):
                continue
            if all(isinstance(getattr(parent, nm, None), nn.Linear) for nm in names):
                plan.setdefault(id(parent), {})[names] = (owner, norm_name, norm)
    return plan


class FusedRMSNorm(nn.Module):
    """An RMSNorm in one launch (rsr_rmsnorm_rows; the BitLinear prologue's
    arithmetic) for bf16 activations -- the norm side of a like-for-like dense
    comparison with fused-norm RSR layers.  Other dtypes use the torch form."""

    def __init__(self, norm: nn.Module):
        super().__init__()
        self.weight = nn.Parameter(norm.weight.data.clone(), requires_grad=False)
        self.variance_epsilon = float(norm.variance_epsilon)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        from . import _lib
        if x.dtype != torch.bfloat16 or self.weight.dtype != torch.bfloat16:
            return rms_norm_reference(x, self.weight, self.variance_epsilon)
        x2 = x.reshape(-1, x.shape[-1]).contiguous()
        out = torch.empty_like(x2)
        _lib.check(_lib.lib().rsr_rmsnorm_rows(x2.data_ptr(), self.weight.data_ptr(), x2.shape[0],
                                               x2.shape[1], self.variance_epsilon,
                                               out.data_ptr(), _lib.current_stream_ptr(x.device)),
                   "rmsnorm")
        return out.view(x.shape)


def fuse_rms_norms(model: nn.Module) -> int:
    """Swap the BitNet decoder layers' RMSNorms (BITNET_NORMS) for
    FusedRMSNorm; returns how many were swapped."""
    count = 0
    for layer in list(model.modules()):
        if not (hasattr(layer, "input_layernorm") and hasattr(layer, "self_attn")):
            continue
        for owner_path, norm_name, _, _ in BITNET_NORMS:
            owner = _sub(layer, owner_path)
            norm = getattr(owner, norm_name, None) if owner is not None else None
            if norm is not None and hasattr(norm, "variance_epsilon"):
                setattr(owner, norm_name, FusedRMSNorm(norm))
                count += 1
    return count


def replace_linear_with_rsr(model: nn.Module, k: int = DEFAULT_K, sibling_groups=DEFAULT_SIBLINGS,
                            skip=("lm_head",), out_dtype=None, fuse_norms: bool = False) -> nn.Module:
    """Replace every bias-free nn.Linear (except `skip`) by an RSRLinear.

    Modeled on transformers' replace_with_bitnet_linear
    (transformers/integrations/bitnet.py:315-370).  Linears named in one
    tuple of `sibling_groups` under the same parent share a stacked artifact.
    The dense weights are released after conversion.

    fuse_norms=True additionally turns each (RMSNorm -> linears) pair of a
    BitNet decoder layer (BITNET_NORMS) into a BitLinear: the norm moves into
    the linears' fused kernel and its module becomes nn.Identity.  Outputs
    equal the unfused layer's up to the fp32 summation order of the norm's
    mean of squares.
    """
    if out_dtype is None:
        out_dtype = next(model.parameters()).dtype
    norms = _norm_plan(model) if fuse_norms else {}
    to_identity = []
    converted = 0
    for parent in list(model.modules()):
        children = dict(parent.named_children())
        pnorms = norms.get(id(parent), {})
        done = set()

        def make_group(names):
            hit = pnorms.get(tuple(names))
            if hit is not None:
                to_identity.append(hit[:2])
            return RSRSiblingGroup([children[nm].weight.data for nm in names], k, out_dtype,
                                   norm=None if hit is None else hit[2])

        for names in sibling_groups:
            if all(isinstance(children.get(nm), nn.Linear) and children[nm].bias is None
                   and nm not in skip for nm in names):
                group = make_group(names)
                for i, nm in enumerate(names):
                    setattr(parent, nm, RSRLinear(group, i))
                    done.add(nm)
                    converted += 1
        for nm, ch in children.items():
            if nm in done or nm in skip or not isinstance(ch, nn.Linear) or ch.bias is not None:
                continue
            group = make_group((nm,))
            setattr(parent, nm, RSRLinear(group, 0))
            converted += 1
    for owner, norm_name in to_identity:
        setattr(owner, norm_name, nn.Identity())
    model._rsr_converted = converted
    model._rsr_fused_norms = len(to_identity)
    torch.cuda.empty_cache()
    return model
