"""Boundary tensors: descriptor + axis-order layout + flat storage.

Same contract as the reference `TensorValue`
(`/root/reference/pkg/src/graphforge/tensor.py:27-125`): `buffer` holds the
elements in *storage* order under `layout`, logical index -> position is
`sum(idx * stride)`, F32 values are kept pre-rounded to binary32.

Storage is a typed buffer instead of a Python list: a 1-D numpy array for
host tensors, or a 1-D CUDA `torch.Tensor` for device-resident tensors (the
B200 path hands those to the kernels without a copy).  torch is used only as
device-memory plumbing.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .errors import RankMismatch
from .ir import ElementType, Shape, TensorDescriptor, element_count
from .layout import Layout, identity_layout

_TORCH_DTYPES = None


def torch_dtype(et: ElementType):
    global _TORCH_DTYPES
    if _TORCH_DTYPES is None:
        import torch

        _TORCH_DTYPES = {
            ElementType.F32: torch.float32,
            ElementType.F64: torch.float64,
            ElementType.I64: torch.int64,
            ElementType.BOOL: torch.bool,
        }
    return _TORCH_DTYPES[et]


def _is_device(buf) -> bool:
    return type(buf).__module__.startswith("torch")


@dataclass
class TensorValue:
    descriptor: TensorDescriptor
    layout: Layout
    buffer: object
    strides: tuple = field(init=False)

    def __post_init__(self):
        if self.layout.rank != len(self.descriptor.shape):
            raise RankMismatch(
                f"layout rank {self.layout.rank} != shape rank {len(self.descriptor.shape)}"
            )
        if len(self.buffer) != self.descriptor.element_count:
            raise RankMismatch(
                f"buffer length {len(self.buffer)} != element count {self.descriptor.element_count}"
            )
        self.strides = self.layout.strides(self.descriptor.shape)

    @property
    def shape(self) -> Shape:
        return self.descriptor.shape

    @property
    def element_type(self) -> ElementType:
        return self.descriptor.element_type

    @property
    def is_device(self) -> bool:
        return _is_device(self.buffer)

    def position(self, index) -> int:
        return sum(i * s for i, s in zip(index, self.strides))

    def _host_storage(self) -> np.ndarray:
        if self.is_device:
            return self.buffer.detach().cpu().numpy()
        return self.buffer

    def get(self, index):
        return self._host_storage()[self.position(index)].item()

    def set(self, index, value) -> None:
        if self.is_device:
            self.buffer[self.position(index)] = value
        else:
            self.buffer[self.position(index)] = coerce_scalar(self.element_type, value)

    def indices(self):
        return itertools.product(*(range(d) for d in self.descriptor.shape))

    def to_numpy(self) -> np.ndarray:
        """Logical row-major contents as an array of `shape`."""
        return storage_to_logical(self._host_storage(), self.shape, self.layout)

    def to_flat(self) -> list:
        return self.to_numpy().reshape(-1).tolist()

    def to_host(self) -> "TensorValue":
        if not self.is_device:
            return self
        return TensorValue(self.descriptor, self.layout, self._host_storage().copy())


def storage_to_logical(storage: np.ndarray, shape, layout: Layout) -> np.ndarray:
    permuted = storage.reshape([shape[a] for a in layout.order])
    inverse = [layout.order.index(i) for i in range(len(shape))]
    return permuted.transpose(inverse)


def logical_to_storage(values: np.ndarray, layout: Layout) -> np.ndarray:
    return np.ascontiguousarray(values.transpose(layout.order)).reshape(-1)


def coerce_array(et: ElementType, data) -> np.ndarray:
    """Row-major values converted the way `coerce_scalar` converts each one."""
    if isinstance(data, np.ndarray):
        arr = data.reshape(-1)
    else:
        arr = np.asarray(list(data) if not isinstance(data, (list, tuple)) else data)
        arr = arr.reshape(-1)
    if et is ElementType.F32:
        if arr.dtype == np.float32:
            return arr.copy()
        with np.errstate(over="ignore", invalid="ignore"):
            return arr.astype(np.float64).astype(np.float32)
    if et is ElementType.F64:
        return arr.astype(np.float64)
    if et is ElementType.I64:
        return arr.astype(np.int64)
    return arr.astype(np.bool_)


def coerce_scalar(et: ElementType, v):
    return coerce_array(et, np.array([v]))[0]


def create_tensor(et: ElementType, shape: Shape, layout: Layout | None = None) -> TensorValue:
    shape = tuple(shape)
    layout = layout or identity_layout(len(shape))
    return TensorValue(TensorDescriptor(et, shape), layout, np.zeros(element_count(shape), dtype=et.numpy_dtype))


def tensor_from_flat(et: ElementType, shape: Shape, data, layout: Layout | None = None) -> TensorValue:
    shape = tuple(shape)
    layout = layout or identity_layout(len(shape))
    values = coerce_array(et, data)
    if values.size != element_count(shape):
        raise RankMismatch(f"data length {values.size} != element count {element_count(shape)}")
    if layout.rank != len(shape):
        raise RankMismatch(f"layout rank {layout.rank} != shape rank {len(shape)}")
    storage = logical_to_storage(values.reshape(shape), layout) if shape else values.copy()
    return TensorValue(TensorDescriptor(et, shape), layout, storage)


def tensor_from_numpy(et: ElementType, array: np.ndarray, layout: Layout | None = None) -> TensorValue:
    return tensor_from_flat(et, array.shape, array, layout)


_BITS = {ElementType.F32: np.uint32, ElementType.F64: np.uint64, ElementType.I64: np.uint64, ElementType.BOOL: np.uint8}


def tensors_bit_equal(a: TensorValue, b: TensorValue) -> bool:
    """Same descriptor and bit-identical logical contents."""
    if a.descriptor != b.descriptor:
        return False
    x = np.ascontiguousarray(a.to_numpy()).reshape(-1)
    y = np.ascontiguousarray(b.to_numpy()).reshape(-1)
    bits = _BITS[a.element_type]
    return bool(np.array_equal(x.view(bits), y.view(bits)))
