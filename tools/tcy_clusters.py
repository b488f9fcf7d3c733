import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1704_06258_b200 as hg  # noqa
inst = hg.generate_urand(1000, 20, 1704, (1.0, 0.75, 1.0))
inst.device()
print("ok")
