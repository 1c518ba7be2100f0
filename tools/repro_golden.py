import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import golden_inputs as gi
import paper_2510_22265_b200 as ebcc
d = json.load(open("tests/golden/chunks.json"))
for i, case in list(enumerate(d["chunks"]))[58:62]:
    a = gi.chunk_input(case)
    print(i, case["kind"], case["rows"], case["cols"], case["eps"], case["q"], case.get("error"), flush=True)
    try:
        b = ebcc.compress(a, case["eps"], case["q"])
        ebcc.decompress(b)
    except ebcc.EbccError as e:
        print("   raised", type(e).__name__, e, flush=True)
