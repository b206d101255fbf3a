import sys
sys.path.insert(0, ".")
from paper_2601_12713_b200 import analyze_columns, savings_columns
from paper_2601_12713_b200.synth import c2_trace
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
c = c2_trace(n)
cf = analyze_columns(c)
sv = savings_columns(c, cf)
print("ok", cf.counts())
