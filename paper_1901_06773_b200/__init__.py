"""B200-native AccUDNN training hot path (arXiv 1901.06773).

Layers:
  * ``planner``  -- Python mirror of the reference ``swapsched`` planner/tuner
    documents API, backed by libswapsched_b200.so (bit-exact host C++).
  * ``kernels``  -- thin ctypes view of the sm_100a layer kernels
    (libaccudnn.so); used by the parity tests.
  * ``trainer``  -- the training-step executor (ResNet on tcgen05 kernels,
    swap executor under a device cap, SGD, NCCL data parallel).
"""

from . import _native  # noqa: F401

__all__ = ["planner", "kernels", "trainer", "resnet_spec"]
