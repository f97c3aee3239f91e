#!/usr/bin/env python3
"""Does a PDL-launched count start before its (triggering) producer ends?
Counts with a mutant library whose griddepcontrol.wait lines are removed,
right behind a slow generator, and compares with the correct library."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
mut = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    f = getattr(mut, name); f.restype = res; f.argtypes = args
n = 256 << 20
buf = torch.zeros(n, dtype=torch.uint8, device="cuda")
c_ok = torch.zeros(16, dtype=torch.int64, device="cuda")
c_mut = torch.zeros(16, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
bad = 0
for i in range(10):
    buf.zero_()
    gen.generate("bernoulli", n, 77 + i, q=30000 + i, out=buf)   # slow ladder generator
    c_mut.zero_()
    _lib.check(mut.pp_count(buf.data_ptr(), n, 16, c_mut.data_ptr(), sp))
    torch.cuda.synchronize()
    c_ok.zero_()
    _lib.check(lib.pp_count(buf.data_ptr(), n, 16, c_ok.data_ptr(), sp))
    torch.cuda.synchronize()
    same = bool((c_ok == c_mut).all())
    bad += not same
    print(i, "same" if same else f"DIFFERENT ok={c_ok[:2].tolist()} mut={c_mut[:2].tolist()}")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pdl in (True,):
    a.record(); gen.generate("bernoulli", n, 5, q=30000, out=buf); t1 = torch.cuda.Event(enable_timing=True); t1.record()
    _lib.check(lib.pp_count(buf.data_ptr(), n, 16, c_ok.data_ptr(), sp)); b.record(); torch.cuda.synchronize()
    print("gen ms", a.elapsed_time(t1), "gen+count ms", a.elapsed_time(b))
print("mismatches", bad)
