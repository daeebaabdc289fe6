timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_disasm.py --modules 200000 --kind disasm
python tools/prof_disasm.py --modules 200000 --kind asm
python tools/phase_disasm.py phases 50000
