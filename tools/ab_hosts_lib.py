"""A/B of the per-host step across library builds (run under gpurun):
VARIANTS="a b" python tools/ab_hosts_lib.py [records] -- one child process per
variant (GNM_LIB=paper_1108_1785_b200/lib/<v>/libgnetmon.so), interleaved,
D3 in HBM, CUDA events around each gnm_analyze call; the row tables' digests
must agree across variants."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    os.execv(sys.executable, [sys.executable, "tools/ab_hosts_median.py", "--child", sys.argv[2]])

n = sys.argv[1] if len(sys.argv) > 1 else "100000000"
for rep in range(int(os.environ.get("ROUNDS", "2"))):
    for v in os.environ["VARIANTS"].split():
        env = dict(os.environ, GNM_LIB=os.path.abspath(f"paper_1108_1785_b200/lib/{v}/libgnetmon.so"),
                   GNM_HOSTS_MEDIAN=v)  # the label printed by the child
        subprocess.run([sys.executable, "tools/ab_hosts_median.py", "--child", n], env=env, check=True)
