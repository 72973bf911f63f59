import sys; sys.path.insert(0, "/root/repo/tools")
from probe_bwd import run
run(8, 32, 8, 8192, 8192, 128, causal=1, time_it=True)
run(8, 32, 8, 8192, 8192, 128, causal=0, time_it=True)
