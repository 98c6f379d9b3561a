"""Runs each alu_peak.cu microbenchmark once (for ncu pipe attribution: run under ncu --metrics sm__inst_executed_pipe_*)."""
import ctypes as C, sys
lib = C.CDLL("paper_2011_09337_b200/libvd_microbench.so")
lib.vdmb_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_double)]
ms, cyc = C.c_float(), C.c_double()
for op in range(11):
    lib.vdmb_run(op, 148*8, 256, 200, C.byref(ms), C.byref(cyc))
