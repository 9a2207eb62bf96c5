"""B200-native core of the Volta GPU-kernel equivalence checker (arXiv 2511.12638).

Product layers: csrc/ (sm_100a CUDA kernels + the C-ABI of include/veq.h,
built in-tree as libveq.so), native.py (ctypes binding), ir.py (packed IR),
engine.py (host mirror of the reference's run()/check reports).
"""
