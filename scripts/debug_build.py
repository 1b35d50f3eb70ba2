import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P
cfg = P.SimConfig(unit_cells=(6, 6, 6), steps=3)
sim = P.Simulation(cfg, mode="fast")
rep = sim.run()
print(rep.thermo)
