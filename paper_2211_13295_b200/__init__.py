"""paper_2211_13295_b200 -- B200-native (sm_100a, FP64) WENO-ADER space-time update.

The product is libhydro_cuda.so (C ABI: include/hydro_cuda.h); ``hydro`` is its Python host
layer mirroring the reference API (proj/include/hydro), ``slabs`` the multi-GPU z-slab driver.
"""
from .hydro import (HLL, OUTFLOW, PERIODIC, RUSANOV, Geom, HostApi, HydroCudaError, Params,
                    Stepper, UnphysicalError, load_library, make_geometry, make_params)

__all__ = ["HLL", "OUTFLOW", "PERIODIC", "RUSANOV", "Geom", "HostApi", "HydroCudaError",
           "Params", "Stepper", "UnphysicalError", "load_library", "make_geometry", "make_params"]
