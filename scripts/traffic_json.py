"""Write profiles/ncu_traffic.json (DRAM read + write bytes per launch of each
bench kernel) from an ncu_summary.py text file.  usage: traffic_json.py SUMMARY"""
import json, re, sys

LABELS = [("k_fbb", "layer0.mm[BMM.FBB]"), ("k_win_bb", "layer0.spmm[BSpMM.BBB]"),
          ("k_sl_gcn1_records", "layer1.mm[BMM.BBF]"), ("k_bv_gcn1", "layer1.spmm[BSpMM.FBF]")]
src = sys.argv[1]
out, cur = {}, None
for line in open(src):
    m = re.match(r"\s*kernel:\s*(.*)", line)
    if m:
        name = m.group(1)
        cur = next((lab for key, lab in LABELS if key in name), None)
        if cur and cur not in out:
            out[cur] = {"kernel": name.split("(")[0].strip(), "source": f"{src} (ncu --set full, one launch)"}
        elif cur:
            cur = None  # first launch of each kernel only
        continue
    m = re.match(r"\s*dram (read|write)\s+([\d.]+) (Mbyte|Gbyte)", line)
    if m and cur:
        out[cur]["dram_" + m.group(1)] = int(round(float(m.group(2)) * (1e9 if m.group(3) == "Gbyte" else 1e6)))
    m = re.match(r"\s*L2->L1 bytes\s+([\d.]+) (Mbyte|Gbyte)", line)
    if m and cur:
        out[cur]["l2_to_l1_bytes"] = int(round(float(m.group(1)) * (1e9 if m.group(2) == "Gbyte" else 1e6)))
for rec in out.values():
    rec["traffic_bytes"] = rec.get("dram_read", 0) + rec.get("dram_write", 0)
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
