import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu
n, E = 6, 4099
Uh = eu.generate_modal_states(E, n, seed=5); Ja = eu.generate_metric(E, n, seed=6)
ss = torch.empty(E, dtype=torch.float64, device="cuda")
R = eu.volume_curvilinear_modal(Uh, Ja, n, sumsq=ss)
torch.save({"R": R.cpu(), "ss": ss.cpu()}, sys.argv[1])
