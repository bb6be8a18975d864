import os, sys
sys.path.insert(0, os.getcwd())
from paper_2103_07925_b200 import scenarios, Simulation
sc = scenarios.config4(T0=1699.7)
sim = Simulation(sc.params, device=0)
sim.upload(sc.store, sc.bodies)
sim.initialize()
sim.step(4)
