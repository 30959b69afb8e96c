"""Print the factor DAG's simulated critical path / makespan (PINLA_VERBOSE line) per config x slots."""
import os, sys
os.environ["PINLA_VERBOSE"] = "1"
sys.path.insert(0, ".")
from paper_2204_04678_b200.objective import ObjectiveEvaluator
from paper_2204_04678_b200.synth import make_instance
for cfg in sys.argv[1:]:
    inst = make_instance(cfg)
    for slots in (1, 3):
        print(f"## {cfg} slots {slots}", file=sys.stderr, flush=True)
        ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=slots)
        ev.close()
