"""Dump SNAP energies/forces of a fixed batch (for comparing kernel variants across processes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_10508_b200 import tungsten as W
q0, box = W.bcc_sia(4)
n = q0.shape[0] // 3
rs = np.random.default_rng(1)
Q = q0[None] + 0.1 * rs.normal(size=(64, q0.shape[0]))
E, G, V = (x.cpu().numpy() for x in W.make_snap(n, box).evaluate(Q, True, True, True))
np.savez(sys.argv[1], E=E, G=G, V=V)
