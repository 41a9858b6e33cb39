"""Head dimensions other than the engine's 64 / 128.

The tcgen05 tiles take D = 64 or 128.  The reference accepts any D (its own tests use
D = 3..8), so the public calls zero-pad the head dimension up to the next engine size
and slice the results back: zero columns change neither Q K^T nor the softmax, they only
add zero columns to O and to the gradients.  The softmax scale stays 1/sqrt(D) of the
caller's D (tensors.py default_scale).  D > 128 raises ShapeError.
"""

import functools

import torch
import torch.nn.functional as F

from .errors import ShapeError
from .tensors import default_scale

__all__ = ["engine_dim", "pad_d", "unpad_d", "padded_call"]


def engine_dim(D):
    """The engine head dim a head dim D runs at."""
    D = int(D)
    if D in (64, 128):
        return D
    if 0 < D < 64:
        return 64
    if 64 < D < 128:
        return 128
    raise ShapeError(f"head dim {D} unsupported (the engine runs D <= 128)")


def pad_d(x, Dp):
    """x (..., D) -> (..., Dp) with zero columns (any tensor / array; result on x's device)."""
    if x is None:
        return None
    t = torch.as_tensor(x)
    D = t.shape[-1]
    if D == Dp:
        return x
    return F.pad(t, (0, Dp - D))


def unpad_d(x, D):
    if x is None or x.shape[-1] == D:
        return x
    return x[..., :D].contiguous()


def _unpad_flash(out, D):
    if out is not None and getattr(out, "O", None) is not None and out.O.shape[-1] != D:
        out.O = unpad_d(out.O, D)
        out._dpad = True
    return out


def _repad_flash(outputs, Dp):
    """FlashOutputs whose O was sliced back to the caller's D, for a backward at Dp."""
    import copy

    if outputs is None or getattr(outputs, "O", None) is None or outputs.O.shape[-1] == Dp:
        return outputs
    o = copy.copy(outputs)
    o.O = pad_d(outputs.O, Dp)
    return o


def padded_call(kind):
    """Decorator for the public calls; `kind` says where the operands and results are."""

    def deco(fn):
        import inspect

        sig = inspect.signature(fn)
        first_name = next(iter(sig.parameters))

        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            x0 = args[0] if args else kwargs[first_name]
            if kind in ("hash_fwd", "hash_bwd"):
                x0 = x0.q
            D = x0.shape[-1] if hasattr(x0, "shape") else torch.as_tensor(x0).shape[-1]
            Dp = engine_dim(D)
            if Dp == D:
                return fn(*args, **kwargs)
            ba = sig.bind(*args, **kwargs)
            ba.apply_defaults()
            a = ba.arguments
            if "scale" in a and a["scale"] is None:
                a["scale"] = default_scale(D)
            if kind in ("attn", "fwd_bwd", "flash_fwd", "flash_bwd", "qk_fwd", "qk_bwd", "prep", "sort"):
                names = [n for n in ("q", "k", "v", "q_c", "k_c", "v_c", "d_out", "d_out_c") if n in a]
                for n in names:
                    a[n] = pad_d(a[n], Dp)
            if kind in ("flash_bwd", "qk_bwd", "hash_bwd"):
                a["outputs"] = _repad_flash(a["outputs"], Dp)
            if kind in ("hash_fwd", "hash_bwd"):
                import copy

                sb = copy.copy(a["sorted_batch"])
                sb.q, sb.k, sb.v = pad_d(sb.q, Dp), pad_d(sb.k, Dp), pad_d(sb.v, Dp)
                a["sorted_batch"] = sb
                if kind == "hash_bwd":
                    a["d_out_sorted"] = pad_d(a["d_out_sorted"], Dp)
            if kind == "fwd_bwd" and a.get("out") is not None:
                out = a["out"]
                a["out"] = None
                res = fn(**a)
                for dst, src in zip(out, res):
                    dst.copy_(unpad_d(src, D))
                return tuple(out)
            res = fn(**a)
            if kind == "attn":
                return unpad_d(res, D)
            if kind in ("fwd_bwd", "flash_bwd", "qk_bwd", "hash_bwd"):
                return tuple(unpad_d(r, D) for r in res)
            if kind in ("flash_fwd", "qk_fwd", "hash_fwd"):
                return _unpad_flash(res, D)
            if kind == "prep":
                return res._replace(q_c=unpad_d(res.q_c, D), k_c=unpad_d(res.k_c, D), v_c=unpad_d(res.v_c, D))
            if kind == "sort":
                res.q, res.k, res.v = unpad_d(res.q, D), unpad_d(res.k, D), unpad_d(res.v, D)
                return res
            return res

        return wrapper

    return deco
