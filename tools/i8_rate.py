"""tcgen05 kind::i8 MMA issue-rate microbenchmark (bem_debug_i8_rate): int8 MACs/s and
cycles per MMA for far10's 21-MMA groups, A in TMEM (TS) or shared memory (SS)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_05186_b200.bem import _check, lib  # noqa: E402

for mode in (0, 1, 2):
    for N in (32, 64, 128, 256):
        r, cy = C.c_double(), C.c_double()
        _check(lib().bem_debug_i8_rate(N, mode, 4000, 0, C.byref(r), C.byref(cy)))
        print(f"mode {['TS', 'SS', 'TS warp'][mode]} N {N:3d}: {r.value / 1e12:8.1f} T int8 MAC/s "
              f"({2 * r.value / 1e12:8.1f} TOP/s), {cy.value:7.1f} cycles per MMA (M128 K32)")
