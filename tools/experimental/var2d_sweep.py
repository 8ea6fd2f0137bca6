import sys; sys.path.insert(0, '.')
import tools.bench_configs as B
for m in (1, 2, 3, 4):
    B.run("cfg3", 2, m, [4096, 4096], boundary=[1, 1], variable=True, steps=10)
