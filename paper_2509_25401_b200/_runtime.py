"""Device plumbing shared by the operators: tensor checks, the device status
word that carries kernel-detected contract violations, and stream handles."""

import torch

from . import _lib
from .errors import DeviceError, ParameterError, ShapeError

TILE = 128  # b_q = b_k = head_dim the sm_100a kernels are built for


def require_cuda():
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 engine has no CPU fallback")
    _lib.load()


def as_device(t, dtype, name):
    """Accept numpy arrays / CPU tensors by copying them to the current device
    once; device tensors of the right dtype pass through untouched."""
    require_cuda()
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    if t.device.type != "cuda":
        t = t.to("cuda")
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def check_bsd(t, name, seq=None, heads=None):
    """[S, H, 128] token-major bf16 activations on the GPU (a [S, H*128] view is
    accepted). The kernels' TMA maps assume a dense row stride of H*128, so a
    strided view (e.g. a head slice q[:, :2]) is copied to a dense tensor."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.bfloat16:
        raise ParameterError(f"{name}: expected a CUDA bf16 tensor")
    if not t.is_contiguous():
        t = t.contiguous()
    if t.dim() == 2:
        if t.shape[1] % TILE:
            raise ShapeError(f"{name}: width {t.shape[1]} not a multiple of {TILE}")
        t = t.view(t.shape[0], t.shape[1] // TILE, TILE)
    if t.dim() != 3:
        raise ShapeError(f"{name}: expected [seq, heads, {TILE}], got {tuple(t.shape)}")
    if t.shape[2] != TILE:
        raise ParameterError(f"{name}: head_dim must be {TILE} for the sm_100a kernels, got {t.shape[2]}")
    if seq is not None and t.shape[0] != seq:
        raise ShapeError(f"{name}: seq {t.shape[0]} != {seq}")
    if heads is not None and t.shape[1] != heads:
        raise ShapeError(f"{name}: heads {t.shape[1]} != {heads}")
    return t


def check_out(t, name, shape, dtype=torch.bfloat16, device=None):
    """Validate a caller-supplied output buffer before a kernel writes into it:
    exact shape, dtype, device and a dense layout (an undersized or strided
    buffer would otherwise be written out of bounds / at the wrong rows)."""
    if not isinstance(t, torch.Tensor):
        raise ParameterError(f"{name}: expected a torch tensor")
    if tuple(t.shape) != tuple(shape) and not (t.numel() == _numel(shape) and t.dim() != len(shape)):
        raise ShapeError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    if t.dtype != dtype:
        raise ParameterError(f"{name}: dtype {t.dtype} != {dtype}")
    if not t.is_cuda or (device is not None and t.device != torch.device(device)):
        raise ParameterError(f"{name}: must live on {device or 'the CUDA device'}, got {t.device}")
    if not t.is_contiguous():
        raise ParameterError(f"{name}: must be contiguous (kernels write a dense row stride)")
    return t


def _numel(shape):
    n = 1
    for s in shape:
        n *= int(s)
    return n


class Status:
    """A uint32 status word in device memory; kernels OR error bits into it."""

    _default = {}

    def __init__(self, device=None):
        self.t = torch.zeros(1, dtype=torch.int32, device=device or "cuda")

    @classmethod
    def default(cls):
        dev = torch.cuda.current_device()
        if dev not in cls._default:
            cls._default[dev] = cls(device=f"cuda:{dev}")
        return cls._default[dev]

    def ptr(self):
        return self.t.data_ptr()

    def check(self, what):
        """Synchronise on the word and raise the reference exception it encodes."""
        bits = int(self.t.item())
        if bits:
            self.t.zero_()
            _lib.raise_status(bits, what)


def check_finite(t, name, status=None, plan=None, what=None, stream=None):
    """Reference as_matrix's finiteness check (tensor.py:19-30) on the device:
    raises ParameterError if `t` (bf16, rows x cols) holds a NaN or Inf. With a
    plan only the active (block, head) tiles are checked (attention.py:194-196).
    Synchronises; called only on the checked (check=True) paths."""
    st = status or Status.default()
    st.check(what or name)  # surface anything already latched under its own name
    rows = t.shape[0]
    cols = t.numel() // max(rows, 1)
    heads = cols // TILE if plan is not None else 0
    _lib.call("fo_check_finite", t.data_ptr(), rows, cols, None if plan is None else plan.ptr(),
              heads, st.ptr(), stream_ptr(stream))
    bits = int(st.t.item())
    if bits:
        st.t.zero_()
        if bits == _lib.ST_PARAM:
            raise ParameterError(f"{name}: contains NaN or Inf")
        _lib.raise_status(bits, what or name)


def stream_ptr(stream=None):
    return _lib.stream_handle(stream)
