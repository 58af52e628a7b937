"""Debug the virtual-rank planner on a small golden case (TIO_LIB_PATH variant)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden, rates_of
from paper_2506_06472_b200 import TransformerGenConfig, gen_transformer_trace
from paper_2506_06472_b200.planner import plan_device_virtual, plan_device
rec = load_golden("c1")[0]
cfg = TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024,
                           bytes_per_element=4, compute_rate=rec["gen"]["compute_rate"], seed=0)
tr = gen_transformer_trace(cfg)
one = plan_device(tr, rec["capacity"], rates_of(rec), rec["host_cap"])
print("single rounds", one["info"].rounds, flush=True)
try:
    outs = plan_device_virtual(tr, rec["capacity"], rates_of(rec), rec["host_cap"], int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    print("virtual ok", [o["plan_bytes"] == one["plan_bytes"] for o in outs])
except Exception as e:
    print("virtual failed", e)
