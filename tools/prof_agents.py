"""cProfile of the agent-mode op mix (tools/bench_agents.py workload, small)."""
import cProfile
import os
import pstats
import sys


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = ["x"] + (sys.argv[1:] or ["--agents", "4", "--rows", "50000", "--rounds", "8"])
import tools.bench_agents as BA  # noqa: E402

cProfile.run("BA.main()", "/tmp/agents.prof")
p = pstats.Stats("/tmp/agents.prof")
p.sort_stats("tottime").print_stats(35)
p.sort_stats("cumulative").print_stats(45)
