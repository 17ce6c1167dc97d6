import ctypes, sys
lib = ctypes.CDLL("tools/libsyncbench.so")
out = (ctypes.c_float * 3)()
for threads, blocks in ((512, 148), (256, 148), (128, 148), (512, 74), (1024, 148)):
    rc = lib.sync_probe(threads, blocks, 2000, out)
    print(threads, blocks, "cg.sync %.2f us  cg.sync+rw %.2f us  custom %.2f us" % tuple(out))
