"""``python -m paper_2603_19371_b200 {synth,register,sweep,membench,reject-ablation}``
(the reference harness CLI)."""
import sys

from .harness import main

sys.exit(main())
