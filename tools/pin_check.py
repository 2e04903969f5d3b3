import ctypes, torch, sys
lib = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "tools/libpincheck.so")
x = torch.empty((1 << 20,), dtype=torch.float32, pin_memory=True)
lib.pin_check(ctypes.c_void_p(x.data_ptr()))
y = torch.empty((1 << 20,), dtype=torch.float32)
lib.pin_check(ctypes.c_void_p(y.data_ptr()))
torch.zeros(1, device="cuda")
lib.pin_check(ctypes.c_void_p(x.data_ptr()))
