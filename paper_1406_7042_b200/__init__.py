"""B200-native hot path of structure-preserving reduced FDTD (arXiv 1406.7042).

* ``fdtd``  - ctypes binding of libfdtd.so (include/fdtd.h), class ``Sim``.
* ``prep``  - host preprocessing library (hybrid assembly, projection basis,
              projection, stability enforcement) producing problem descriptions.
* ``build`` - compiles libfdtd.so for sm_100a in-tree.
"""
__version__ = "0.1.0"
