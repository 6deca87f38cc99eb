import sys, os, warnings
warnings.simplefilter("ignore")
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2206_11357_b200 as gact
from paper_2206_11357_b200.controller import Controller

def mlp(widths, act=torch.nn.Tanh, seed=0):
    torch.manual_seed(seed)
    layers = []
    for a, b in zip(widths[:-1], widths[1:]):
        layers += [torch.nn.Linear(a, b), act()]
    return torch.nn.Sequential(*layers[:-1]).cuda()

def run(avg, cseed, lr=0.05):
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.randn(16, 64, device="cuda", generator=g) * 1.5
    m = mlp([64, 512, 512, 16], act=torch.nn.ReLU, seed=1)
    opt = torch.optim.SGD(m.parameters(), lr=lr, momentum=0.9)
    c = None if avg is None else Controller(m, avg_bits=avg, ladder=(1, 2, 4, 8), merge=False, adapt_interval=100, seed=cseed)
    hist = []
    for it in range(300):
        y = torch.randint(0, 16, (512,), device="cuda", generator=g)
        x = centers[y] + torch.randn(512, 64, device="cuda", generator=g)
        def f():
            loss = torch.nn.functional.cross_entropy(m(x), y)
            loss.backward()
            f.loss = float(loss)
        try:
            if c is None:
                opt.zero_grad(); f()
            else:
                c.iterate(f)
        except Exception as e:
            return f"diverged at {it}", hist
        opt.step()
        if it in (99, 150, 199, 250, 299): hist.append(round(f.loss, 4))
    y = torch.randint(0, 16, (512,), device="cuda", generator=g)
    x = centers[y] + torch.randn(512, 64, device="cuda", generator=g)
    with torch.no_grad():
        acc = float((m(x).argmax(1) == y).float().mean())
    return acc, (hist, None if c is None else c.bits)

tag = os.environ.get("GACT_LIB_PATH", "new")
for lr in [0.02, 0.01]:
    print(tag, lr, "fp32", run(None, 0, lr))
    for s in [3, 4, 5, 6, 7, 8]:
        print(tag, lr, 2, s, run(2, s, lr))
