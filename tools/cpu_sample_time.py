import sys, time
sys.path.insert(0, ".")
import bench
t0 = time.perf_counter()
import oracle as O
a = O.generate_test_matrix("lu", int(sys.argv[1]), 0)
print("gen", time.perf_counter() - t0, flush=True)
for it in (1,):
    print(bench.cpu_sample("lu", int(sys.argv[1]), 256, "full", 0, it, a), flush=True)
