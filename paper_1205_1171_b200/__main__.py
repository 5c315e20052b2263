"""python -m paper_1205_1171_b200 {generate,hull,verify,bench} ..."""
from .cli import main_entry

main_entry()
