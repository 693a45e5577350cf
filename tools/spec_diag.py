"""Where speculative and plain greedy decoding diverge: oracle margin there."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from oracle.model import init_weights_llama, llama_tiny_config
from helpers import c1_prompts, device_weights
from paper_2507_11830_b200 import Engine, LoopbackGroup, ShiftPolicy
from paper_2507_11830_b200.spec_decode import SpeculationConfig, decode_with_speculation

c1 = init_weights_llama(llama_tiny_config(max_seq=512), seed=0)
eng = Engine(device_weights(c1, 1), LoopbackGroup(1), ShiftPolicy(token_threshold=3))
prompt = [11, 42, 7, 99, 3] * 6 + c1_prompts()[2][:17]
plain, _ = decode_with_speculation(eng, prompt, 40, SpeculationConfig(enabled=False))
spec, st = decode_with_speculation(eng, prompt, 40, SpeculationConfig(enabled=True, min_match=1, max_spec=6))
print("plain", plain)
print("spec ", spec)
print("accepted", st.accepted_lengths)
i = next((k for k in range(40) if plain[k] != spec[k]), None)
print("first diff", i)
if i is not None:
    lg, _ = oracle.forward_reference(c1, prompt + plain[:i])
    row = lg[-1]
    o = np.argsort(-row)[:4]
    print("oracle top4", [(int(t), float(row[t])) for t in o], "plain", plain[i], row[plain[i]], "spec", spec[i], row[spec[i]])
