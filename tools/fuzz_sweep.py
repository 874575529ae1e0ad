"""Large randomised sweep (B200): the three generators of tests/test_gpu_fuzz.py with many more cases
and another seed -- oracle parity of random chains, bit-identity across engine knobs, stage splits.
    python tools/fuzz_sweep.py SEED            (profiles/r02_fuzz_sweep.txt)"""
import sys, time, traceback
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu_fuzz as F
t0 = time.time()
fails = []
sets = [(F._cases(3000, seed=int(sys.argv[1])), F.test_random_chain_vs_oracle),
        (F._knob_cases(1500, seed=int(sys.argv[1]) + 1), F.test_random_knobs_bit_identical),
        (F._split_cases(800, seed=int(sys.argv[1]) + 2), F.test_random_stage_split_equals_full_chain)]
for cases, fn in sets:
    for c in cases:
        try:
            fn(c)
        except Exception as e:
            fails.append((fn.__name__, c, repr(e)[:300]))
    print(fn.__name__, len(cases), "cases, fails so far", len(fails), "t=%.0fs" % (time.time() - t0), flush=True)
for f in fails[:10]:
    print("FAIL", f)
