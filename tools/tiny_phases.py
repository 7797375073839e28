import sys
sys.path.insert(0, '/root/repo')
import paper_2604_16613_b200 as gp
g = gp.gen_surface(3, 3, 1e-3)
comp = gp.Compiler(0)
for _ in range(50): comp.compile(g, 0)
comp.set_option(99, 4)
for _ in range(5): comp.compile(g, 0)
