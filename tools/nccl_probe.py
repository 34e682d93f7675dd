"""Probe: open libnccl through the product library and build a communicator
over the visible devices (bmc_nccl_init_all).  Diagnostic only."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27193_b200 as bmc  # noqa: E402

lib = bmc.load()
v = C.c_int(0)
rc = lib.bmc_nccl_available(C.byref(v))
print("available rc", rc, "version", v.value, lib.bmc_last_error())
n = bmc.device_count()
devs = (C.c_int * n)(*range(n))
comms = (C.c_void_p * n)()
rc = lib.bmc_nccl_init_all(n, devs, comms)
print("init_all rc", rc, lib.bmc_last_error())
