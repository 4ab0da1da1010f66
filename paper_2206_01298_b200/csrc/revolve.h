#pragma once
#include <vector>

namespace ob {

enum ActionKind { kAdvance = 0, kStore = 1, kRestore = 2, kReverse = 3 };

struct Action {
  int kind, step, start, stop;
};

long long revolve_count(int nt, int nc);
std::vector<Action> revolve_schedule(int nt, int nc);

}  // namespace ob
