# run the C++ shim parity binary on the golden graphs (debug helper)
mkdir -p /tmp/gg && python - <<'PY'
import json
g = json.load(open("tests/golden/golden.json"))
for r in g["graphs"]:
    open(f"/tmp/gg/{r['name']}.json", "w").write(r["graph_json"])
PY
tests/cpp/_bin/shim_parity /tmp/gg/*.json 2>&1 | sort | uniq -c | sort -rn | head -20
