import os, sys
sys.path.insert(0, "/root/repo")
os.environ["EI_PLAN_VERBOSE"] = "1"
from paper_2202_08627_b200 import ei, synth
for c in ["C1", "C2", "C3", "C4", "C5"]:
    cfg = synth.CONFIGS[c]
    pl = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
    print(c, ei.ei_plan_info(pl), flush=True)
