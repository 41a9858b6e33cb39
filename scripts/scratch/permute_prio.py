"""cfg2: K/V permute concurrent with the schedule build, with stream priorities (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from permute_iso import timeit, k, v, rank, B, T, H, D, dev, sched, hs

lo = torch.cuda.Stream(dev, priority=0)
hi = torch.cuda.Stream(dev, priority=-5)
print("priority range", torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else None,
      "hi", hi.priority, "lo", lo.priority)
print(f"sched alone again: {timeit(sched):.1f} us")
def both_hi():
    main = torch.cuda.current_stream()
    lo.wait_stream(main); hi.wait_stream(main)
    with torch.cuda.stream(lo):
        hs._permute3([k, v], [rank, rank], T)
    with torch.cuda.stream(hi):
        sched()
    main.wait_stream(lo); main.wait_stream(hi)
print(f"permute(lo) || sched(hi): {timeit(both_hi):.1f} us")
def both_hi_first():
    main = torch.cuda.current_stream()
    lo.wait_stream(main); hi.wait_stream(main)
    with torch.cuda.stream(hi):
        sched()
    with torch.cuda.stream(lo):
        hs._permute3([k, v], [rank, rank], T)
    main.wait_stream(lo); main.wait_stream(hi)
print(f"sched(hi) first || permute(lo): {timeit(both_hi_first):.1f} us")
def perm_hi():
    main = torch.cuda.current_stream()
    hi.wait_stream(main)
    with torch.cuda.stream(hi):
        hs._permute3([k, v], [rank, rank], T)
    sched()
    main.wait_stream(hi)
print(f"permute(hi) || sched(main): {timeit(perm_hi):.1f} us")
