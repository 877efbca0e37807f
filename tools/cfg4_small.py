import sys; sys.path.insert(0, '.')
import torch
from paper_1806_01422_b200 import configs
prob = configs.cfg4_problem(B=512, steps=50, device="cuda:0")
j, g = prob.evaluate(prob.u_guess)
torch.cuda.synchronize()
print("ok")
